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

// grid for an (nx, ny, nz) local block: (z tiles, y tiles, x chunks)
inline bool stencil7_grid(int64_t nx, int64_t ny, int64_t nz, int64_t xchunk, dim3& grid) {
  const int64_t gz = (nz + kTileZ - 1) / kTileZ;
  const int64_t gy = (ny + kTileY - 1) / kTileY;
  const int64_t gx = (nx + xchunk - 1) / xchunk;
  if (gz > INT32_MAX || gy > 65535 || gx > 65535) return false;
  grid = dim3(static_cast<unsigned>(gz), static_cast<unsigned>(gy), static_cast<unsigned>(gx));
  return true;
}

}  // namespace kls
