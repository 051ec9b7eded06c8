// TMA-staged 7-point stencil (the default for 16-byte-aligned grids): the
// CTA owns a 64 (z) x 16 (y) tile and marches an x-chunk; a producer warp
// streams each plane's tile plus its one-point y / z halo (18 rows of 68
// doubles, z0-2 .. z0+66, 16-byte aligned) into a 4-stage shared-memory
// ring -- ONE 3-D tensor copy per plane (cp.async.bulk.tensor on a
// cuTensorMapEncodeTiled map of the rank's block; the hardware zero-fills
// the box outside the grid), or 18 row copies (cp.async.bulk) without a
// tensor map -- so ~3 planes per CTA are in flight independently of
// registers.  The register-marching kernels kept 16 B per thread in flight
// and reached 4.45 TB/s (ncu: DRAM 53 %); 544-byte row copies alone gave
// the same rate (small bulk copies), hence the tensor map.
// 8 consumer warps compute 4 points each per plane (z = lane, lane + 32;
// y = warp, warp + 8) with the x-1 / x / x+1 centres in registers and the
// y / z neighbours from the ring, in the reference's order (6 g, then minus
// x-1, x+1, y-1, y+1, z-1, z+1, explicitly rounded): bit-identical to
// StencilLaplace3D._matvec (problems.py:296-305) and the other variants.
// Rank-boundary planes (x_lo / x_hi, another GPU's memory) are copied into
// the ring by the consumer threads with coherent loads after the
// neighbour's halo flag (peer kernel) -- the same kernel serves both.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "peer.cuh"
#include "stencil.cuh"
#include "tma.cuh"

namespace kls {

constexpr int kTZ = 64, kTY = 16;          // tile
constexpr int kRowD = kTZ + 4;             // ring row: z0-2 .. z0+66 (68 doubles)
constexpr int kRowsS = kTY + 2;            // ring rows per stage: y0-1 .. y0+16
constexpr int kStageD = kRowsS * kRowD;    // doubles per stage (the TMA box)
constexpr int kStageStride = (kStageD + 15) / 16 * 16;  // 128-byte aligned stages
constexpr int kTStages = 4;
constexpr int kTThreads = 9 * 32;          // 8 consumer warps + 1 producer warp

struct TmaStencilArgs {
  int32_t use_map;     // the tensor map below describes x (local planes)
  const double* x;
  const double* x_lo;  // neighbouring planes (other ranks) or nullptr
  const double* x_hi;
  double* y;
  int64_t nx;
  int32_t ny, nz, xchunk;
  // peer halo flags (kls_stencil7_peer); nullptr: no waiting
  const uint64_t* flag_lo;
  const uint64_t* flag_hi;
  uint64_t epoch;
  int* err;
};

__device__ __forceinline__ void tensor3d_g2s(void* dst, const CUtensorMap* map, int c0, int c1,
                                             int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(tma::su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(tma::su32(bar))
      : "memory");
}

static __global__ void __launch_bounds__(kTThreads) stencil7_tma_kernel(
    const TmaStencilArgs a, const __grid_constant__ CUtensorMap map) {
  using namespace kls::tma;
  __shared__ __align__(128) double ring[kTStages][kStageStride];
  __shared__ __align__(8) uint64_t full[kTStages], empty[kTStages];
  __shared__ int s_ok;
  pdl_wait();  // x from the preceding update
  const int64_t xa = static_cast<int64_t>(blockIdx.z) * a.xchunk;
  const int64_t xb = xa + a.xchunk < a.nx ? xa + a.xchunk : a.nx;
  if (xa >= xb) return;  // uniform per CTA
  const int32_t z0 = blockIdx.x * kTZ, y0 = blockIdx.y * kTY;
  const int64_t plane = static_cast<int64_t>(a.ny) * a.nz;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // planes xa-1 .. xb, of which the ones outside [0, nx) come from x_lo /
  // x_hi (copied by the consumers) or are absent (Dirichlet boundary)
  const bool lo_halo = xa == 0 && a.x_lo != nullptr;
  const bool hi_halo = xb == a.nx && a.x_hi != nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_ok = 1;
    if (lo_halo && a.flag_lo != nullptr && !peer::wait_flag(a.flag_lo, a.epoch)) s_ok = 0;
    if (hi_halo && a.flag_hi != nullptr && !peer::wait_flag(a.flag_hi, a.epoch)) s_ok = 0;
    if (!s_ok && a.err != nullptr) *a.err = 1;
  }
  __syncthreads();
  if (!s_ok) return;
  const int zs = z0 - 2 > 0 ? z0 - 2 : 0;
  const int ze = z0 + kTZ + 2 < a.nz ? z0 + kTZ + 2 : a.nz;
  const int ys = y0 - 1 > 0 ? y0 - 1 : 0;
  const int ye = y0 + kTY + 1 < a.ny ? y0 + kTY + 1 : a.ny;
  const int zoff = zs - (z0 - 2);
  const int nplanes = static_cast<int>(xb - xa) + 2;  // xa-1 .. xb
  if (warp == 8) {  // producer: one elected lane issues the bulk copies
    if (lane == 0) {
      const uint32_t rbytes = static_cast<uint32_t>(ze - zs) * sizeof(double);
      for (int q = 0; q < nplanes; ++q) {
        const int s = q % kTStages;
        if (q >= kTStages) mbar_wait(empty + s, ((q / kTStages) - 1) & 1);
        const int64_t px = xa - 1 + q;
        if (px < 0 || px >= a.nx) {  // halo plane (consumers fill) or absent
          mbar_arrive(full + s);
          continue;
        }
        if (a.use_map) {  // the whole box, out-of-grid elements zero-filled
          mbar_expect_tx(full + s, kStageD * sizeof(double));
          tensor3d_g2s(ring[s], &map, z0 - 2, y0 - 1, static_cast<int>(px), full + s);
          continue;
        }
        mbar_expect_tx(full + s, rbytes * static_cast<uint32_t>(ye - ys));
        const double* src = a.x + px * plane + zs;
        for (int yy = ys; yy < ye; ++yy)
          bulk_g2s(ring[s] + (yy - (y0 - 1)) * kRowD + zoff, src + static_cast<int64_t>(yy) * a.nz,
                   rbytes, full + s);
      }
    }
    return;
  }
  // consumer: 4 points (z = lane, lane + 32; y = warp, warp + 8)
  const int tid = threadIdx.x;  // 0..255
  int32_t iz[2], iy[2];
  bool ok[2][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    iz[c] = z0 + lane + 32 * c;
    iy[c] = y0 + warp + 8 * c;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int c = 0; c < 2; ++c) ok[r][c] = iy[r] < a.ny && iz[c] < a.nz;
  auto at = [&](int s, int ry, int cz) -> double {  // ring value at tile row ry, column cz
    return ring[s][(ry + 1) * kRowD + cz + 2];
  };
  // a halo plane from another rank: the consumers copy its tile (+ y/z halo)
  auto fill_halo = [&](int s, const double* src) {
    const int w = ze - zs;
    for (int i = tid; i < (ye - ys) * w; i += 256) {
      const int yy = ys + i / w, zz = zs + i % w;
      ring[s][(yy - (y0 - 1)) * kRowD + (zz - (z0 - 2))] =
          ld_halo(src + static_cast<int64_t>(yy) * a.nz + zz);
    }
    // generic writes into a stage the bulk copies may refill later
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 256;" ::: "memory");
  };
  double prv[2][2], cur[2][2], nxt[2][2];
  // planes xa-1 (q = 0) and xa (q = 1)
  for (int q = 0; q < 2; ++q) {
    const int s = q % kTStages;
    mbar_wait(full + s, 0);
    const int64_t px = xa - 1 + q;
    if (px < 0 && lo_halo) fill_halo(s, a.x_lo);
    if (px >= a.nx && hi_halo) fill_halo(s, a.x_hi);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double v = at(s, warp + 8 * r, lane + 32 * c);
        if (q == 0) prv[r][c] = v; else cur[r][c] = v;
      }
  }
  // plane xa-1 lives on in registers only
  __syncwarp();
  if (lane == 0) mbar_arrive(empty + 0);
  for (int q = 2; q < nplanes; ++q) {  // output plane xa-2+q uses planes q-2, q-1, q
    const int s = q % kTStages, sc = (q - 1) % kTStages;
    mbar_wait(full + s, (q / kTStages) & 1);
    const int64_t px = xa - 1 + q;
    if (px >= a.nx && hi_halo) fill_halo(s, a.x_hi);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) nxt[r][c] = at(s, warp + 8 * r, lane + 32 * c);
    const int64_t ox = px - 1;  // the output plane
    const bool hp = ox > 0 || a.x_lo != nullptr;
    const bool hn = ox + 1 < a.nx || a.x_hi != nullptr;
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        if (!ok[r][c]) continue;
        const int ry = warp + 8 * r, cz = lane + 32 * c;
        double acc = __dmul_rn(6.0, cur[r][c]);
        if (hp) acc = __dsub_rn(acc, prv[r][c]);
        if (hn) acc = __dsub_rn(acc, nxt[r][c]);
        if (iy[r] > 0) acc = __dsub_rn(acc, at(sc, ry - 1, cz));
        if (iy[r] + 1 < a.ny) acc = __dsub_rn(acc, at(sc, ry + 1, cz));
        if (iz[c] > 0) acc = __dsub_rn(acc, at(sc, ry, cz - 1));
        if (iz[c] + 1 < a.nz) acc = __dsub_rn(acc, at(sc, ry, cz + 1));
        a.y[ox * plane + static_cast<int64_t>(iy[r]) * a.nz + iz[c]] = acc;
      }
    // plane q-1's stage (this output's y / z neighbours) is done
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + sc);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        prv[r][c] = cur[r][c];
        cur[r][c] = nxt[r][c];
      }
  }
  pdl_trigger();
}

// eligibility: 16-byte aligned rows (nz even, x aligned)
inline bool stencil7_tma_ok(const double* x, int64_t ny, int64_t nz) {
  return (nz % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 && ny <= 65535 * kTY &&
         nz <= INT32_MAX;
}

// The 3-D tensor map of a rank's block x (nx planes of ny x nz, z fastest)
// with the ring's box (68 x 18 x 1); false when the driver entry point or
// the encode is unavailable (the kernel then issues row copies).  Maps are
// cached per (x, shape).
bool stencil7_tensor_map(const double* x, int64_t nx, int64_t ny, int64_t nz, CUtensorMap* map);

}  // namespace kls
