// The 7-point stencil march shared by kls_stencil7 and kls_stencil7_peer.
//
// CTA = a 32 (z) x 8 (y) tile of lines marching through a chunk of x-planes.
// Each thread keeps its line's x-1 / x / x+1 values in registers (every
// element is read from HBM once); the y+-1 and z+-1 neighbours are the
// centres of other threads of the same CTA in the same plane, so they hit
// L1 except on the tile border (2 of 8 rows, 2 of 32 columns).  The sum is
// formed exactly as StencilLaplace3D._matvec (problems.py:296-305):
// 6 g, then minus x-1, x+1, y-1, y+1, z-1, z+1, each an explicitly rounded
// __dmul_rn / __dsub_rn.
#pragma once

#include "common.cuh"

namespace kls {

constexpr int kTileZ = 32;
constexpr int kTileY = 8;

// halo planes of another rank: coherent loads (written before the flag)
__device__ __forceinline__ double ld_halo(const double* p) {
  return *reinterpret_cast<const volatile double*>(p);
}

// one output: 6 g - x-1 - x+1 - y-1 - y+1 - z-1 - z+1 in the reference order
__device__ __forceinline__ double stencil7_point(const double* __restrict__ x, int64_t i, double g,
                                                 bool hp, double p, bool hn, double n, bool ylo,
                                                 bool yhi, bool zlo, bool zhi, int32_t nz) {
  double acc = __dmul_rn(6.0, g);
  if (hp) acc = __dsub_rn(acc, p);
  if (hn) acc = __dsub_rn(acc, n);
  if (ylo) acc = __dsub_rn(acc, __ldg(x + i - nz));
  if (yhi) acc = __dsub_rn(acc, __ldg(x + i + nz));
  if (zlo) acc = __dsub_rn(acc, __ldg(x + i - 1));
  if (zhi) acc = __dsub_rn(acc, __ldg(x + i + 1));
  return acc;
}

// Marches a line through planes [xa, xb) in groups of kG: the kG upcoming
// planes are loaded together (kG independent HBM loads in flight per
// thread), then kG outputs are formed from the register window.
__device__ __forceinline__ void stencil7_march(const double* __restrict__ x,
                                               const double* x_lo, const double* x_hi,
                                               double* __restrict__ y, int64_t nx, int32_t ny,
                                               int32_t nz, int64_t xa, int64_t xb) {
  constexpr int kG = 4;
  const int32_t iz = blockIdx.x * kTileZ + threadIdx.x;
  const int32_t iy = blockIdx.y * kTileY + threadIdx.y;
  if (iz >= nz || iy >= ny || xa >= xb) return;
  const int64_t plane = static_cast<int64_t>(ny) * nz;
  const int64_t t = static_cast<int64_t>(iy) * nz + iz;
  const bool ylo = iy > 0, yhi = iy + 1 < ny, zlo = iz > 0, zhi = iz + 1 < nz;
  bool hp = xa > 0 || x_lo != nullptr;
  double prev = xa > 0 ? __ldg(x + (xa - 1) * plane + t) : (x_lo != nullptr ? ld_halo(x_lo + t) : 0.0);
  double cur = __ldg(x + xa * plane + t);
  int64_t ix = xa;
  for (; ix + kG <= xb; ix += kG) {
    double w[kG];  // planes ix+1 .. ix+kG
    bool hv[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      const int64_t jx = ix + 1 + g;
      hv[g] = jx < nx || x_hi != nullptr;
      w[g] = jx < nx ? __ldg(x + jx * plane + t) : (x_hi != nullptr ? ld_halo(x_hi + t) : 0.0);
    }
    double out[kG];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      const double c = g == 0 ? cur : w[g - 1];
      const double p = g == 0 ? prev : (g == 1 ? cur : w[g - 2]);
      const bool hpg = g == 0 ? hp : true;
      out[g] = stencil7_point(x, (ix + g) * plane + t, c, hpg, p, hv[g], w[g], ylo, yhi, zlo, zhi, nz);
    }
#pragma unroll
    for (int g = 0; g < kG; ++g) y[(ix + g) * plane + t] = out[g];
    prev = w[kG - 2];
    cur = w[kG - 1];
    hp = true;
  }
  for (; ix < xb; ++ix) {
    const int64_t i = ix * plane + t;
    const bool hn = ix + 1 < nx || x_hi != nullptr;
    const double next = ix + 1 < nx ? __ldg(x + i + plane) : (x_hi != nullptr ? ld_halo(x_hi + t) : 0.0);
    y[i] = stencil7_point(x, i, cur, hp, prev, hn, next, ylo, yhi, zlo, zhi, nz);
    prev = cur;
    cur = next;
    hp = true;
  }
}

// Shared-memory variant: the CTA owns a 64 (z) x 8 (y) tile (lane l handles
// z = l and l + 32, one warp per y row: conflict-free shared-memory rows) and marches through its x-chunk keeping the current
// plane's tile plus a one-point halo in shared memory and the x-1 / x / x+1
// values of its own points in registers.  Each plane's tile is read from
// global memory once (the y / z halo rows come from L2); the next plane's
// loads are issued a full iteration before they are used.
constexpr int kSTZ = 64;
constexpr int kSTY = 8;

__device__ __forceinline__ double ld_plane(const double* __restrict__ x, const double* x_lo,
                                           const double* x_hi, int64_t ix, int64_t nx,
                                           int64_t plane, int64_t t) {
  if (ix >= 0 && ix < nx) return __ldg(x + ix * plane + t);
  if (ix < 0) return x_lo != nullptr ? ld_halo(x_lo + t) : 0.0;
  return x_hi != nullptr ? ld_halo(x_hi + t) : 0.0;
}

__device__ __forceinline__ void stencil7_tile_march(const double* __restrict__ x,
                                                    const double* x_lo, const double* x_hi,
                                                    double* __restrict__ y, int64_t nx, int32_t ny,
                                                    int32_t nz, int64_t xa, int64_t xb,
                                                    double (*tile)[kSTZ + 2]) {
  const int lx = threadIdx.x, ly = threadIdx.y;
  const int32_t z0 = blockIdx.x * kSTZ, y0 = blockIdx.y * kSTY;
  const int32_t iy = y0 + ly;
  const int32_t iz[2] = {z0 + lx, z0 + lx + 32};
  const int64_t plane = static_cast<int64_t>(ny) * nz;
  const bool row_ok = iy < ny;
  bool ok[2];
  int64_t t[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    ok[c] = row_ok && iz[c] < nz;
    t[c] = static_cast<int64_t>(iy) * nz + iz[c];
  }
  // halo roles: warp 0 loads the row below the tile, warp 7 the row above,
  // lanes 0 / 31 the z columns left / right of their row
  const int32_t hy = ly == 0 ? y0 - 1 : (ly == kSTY - 1 ? y0 + kSTY : -1);
  const bool hy_ok = hy >= 0 && hy < ny;
  const int32_t hz = lx == 0 ? z0 - 1 : (lx == 31 ? z0 + kSTZ : -1);
  const bool hz_ok = row_ok && hz >= 0 && hz < nz;
  auto load_halo = [&](int64_t ix, double (&hrow)[2], double& hcol) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
      hrow[c] = (hy_ok && iz[c] < nz)
                    ? ld_plane(x, x_lo, x_hi, ix, nx, plane, static_cast<int64_t>(hy) * nz + iz[c])
                    : 0.0;
    hcol = hz_ok ? ld_plane(x, x_lo, x_hi, ix, nx, plane, static_cast<int64_t>(iy) * nz + hz) : 0.0;
  };
  auto store_tile = [&](const double (&core)[2], const double (&hrow)[2], double hcol) {
    tile[ly + 1][lx + 1] = core[0];
    tile[ly + 1][lx + 33] = core[1];
    if (ly == 0) {
      tile[0][lx + 1] = hrow[0];
      tile[0][lx + 33] = hrow[1];
    }
    if (ly == kSTY - 1) {
      tile[kSTY + 1][lx + 1] = hrow[0];
      tile[kSTY + 1][lx + 33] = hrow[1];
    }
    if (lx == 0) tile[ly + 1][0] = hcol;
    if (lx == 31) tile[ly + 1][kSTZ + 1] = hcol;
  };
  const bool has_lo = x_lo != nullptr, has_hi = x_hi != nullptr;
  double prv[2], cur[2], nxt[2], hrow[2], hcol;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    prv[c] = ok[c] ? ld_plane(x, x_lo, x_hi, xa - 1, nx, plane, t[c]) : 0.0;
    cur[c] = ok[c] ? ld_plane(x, x_lo, x_hi, xa, nx, plane, t[c]) : 0.0;
    nxt[c] = ok[c] ? ld_plane(x, x_lo, x_hi, xa + 1, nx, plane, t[c]) : 0.0;
  }
  load_halo(xa, hrow, hcol);
  store_tile(cur, hrow, hcol);
  const bool ylo = iy > 0, yhi = iy + 1 < ny;
  for (int64_t ix = xa; ix < xb; ++ix) {
    // loads for later: own points of plane ix+2, halo of plane ix+1
    double nn[2], nhrow[2], nhcol = 0.0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      nn[c] = (ok[c] && ix + 1 < xb) ? ld_plane(x, x_lo, x_hi, ix + 2, nx, plane, t[c]) : 0.0;
      nhrow[c] = 0.0;
    }
    if (ix + 1 < xb) load_halo(ix + 1, nhrow, nhcol);
    __syncthreads();  // the tile holds plane ix
    const bool hp = ix > 0 || has_lo;
    const bool hn = ix + 1 < nx || has_hi;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (!ok[c]) continue;
      const int sz = lx + 1 + 32 * c;
      double acc = __dmul_rn(6.0, cur[c]);
      if (hp) acc = __dsub_rn(acc, prv[c]);
      if (hn) acc = __dsub_rn(acc, nxt[c]);
      if (ylo) acc = __dsub_rn(acc, tile[ly][sz]);
      if (yhi) acc = __dsub_rn(acc, tile[ly + 2][sz]);
      if (iz[c] > 0) acc = __dsub_rn(acc, tile[ly + 1][sz - 1]);
      if (iz[c] + 1 < nz) acc = __dsub_rn(acc, tile[ly + 1][sz + 1]);
      y[ix * plane + t[c]] = acc;
    }
    __syncthreads();  // everyone is done with plane ix
    if (ix + 1 < xb) store_tile(nxt, nhrow, nhcol);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      prv[c] = cur[c];
      cur[c] = nxt[c];
      nxt[c] = nn[c];
    }
  }
}

// grid for an (nx, ny, nz) local block: (z tiles, y tiles, x chunks)
inline bool stencil7_grid(int64_t nx, int64_t ny, int64_t nz, int64_t xchunk, dim3& grid,
                          int tz = kTileZ, int ty = kTileY) {
  const int64_t gz = (nz + tz - 1) / tz;
  const int64_t gy = (ny + ty - 1) / ty;
  const int64_t gx = (nx + xchunk - 1) / xchunk;
  if (gz > INT32_MAX || gy > 65535 || gx > 65535) return false;
  grid = dim3(static_cast<unsigned>(gz), static_cast<unsigned>(gy), static_cast<unsigned>(gx));
  return true;
}

}  // namespace kls
