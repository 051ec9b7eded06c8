// Deterministic grid-wide reduction of a few per-thread accumulators.
//
// Every CTA reduces its threads (warp shuffles, then warps in index order),
// writes one partial per value to a workspace, and the last CTA to arrive
// (atomic ticket) sums the partials in CTA order.  No fp64 atomics, so the
// result is bitwise reproducible for a fixed grid.
#pragma once

#include "common.cuh"

namespace kls {

constexpr size_t kTicketBytes = 256;

struct RedWs {
  unsigned int* ticket;
  double* partials;
};

inline RedWs red_ws(void* ws) {
  RedWs r;
  r.ticket = static_cast<unsigned int*>(ws);
  r.partials = reinterpret_cast<double*>(static_cast<char*>(ws) + kTicketBytes);
  return r;
}

inline bool red_ws_fits(size_t ws_bytes, int grid, int nv) {
  return kTicketBytes + static_cast<size_t>(grid) * nv * sizeof(double) <= ws_bytes;
}

// Fixed-order sum over the nb CTA partials (row stride nv) of every entry,
// by the whole (last) CTA: entry i is summed by S threads, thread s taking
// CTAs b = s, s+S, ... into 8 independent accumulators (8 loads in flight),
// and the S slice sums are added in slice order through shared memory.
// emit(i, sum) is called once per entry.  Must be reached by every thread.
template <typename Emit>
__device__ __forceinline__ void sum_partials_block(const double* partials, int nb, int nv,
                                                   Emit emit) {
  __shared__ double s_red[512];
  const int T = blockDim.x;
  int S = nv > 0 ? T / nv : 1;
  S = S >= 16 ? 16 : S >= 8 ? 8 : S >= 4 ? 4 : S >= 2 ? 2 : 1;
  const int per_round = T / S;
  const int slot = threadIdx.x / S;
  const int sl = threadIdx.x % S;
  for (int base = 0; base < nv; base += per_round) {
    const int i = base + slot;
    const bool live = slot < per_round && i < nv;
    double v = 0.0;
    if (live) {
      double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int b = sl;
      for (; b + 7 * S < nb; b += 8 * S) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += __ldcg(partials + static_cast<int64_t>(b + u * S) * nv + i);
      }
      for (; b < nb; b += S) a[0] += __ldcg(partials + static_cast<int64_t>(b) * nv + i);
      v = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    s_red[threadIdx.x] = v;
    __syncthreads();
    if (live && sl == 0) {
      double t = 0.0;
      for (int k = 0; k < S; ++k) t += s_red[threadIdx.x + k];
      emit(i, t);
    }
    __syncthreads();
  }
}

// Must be reached by every thread of every CTA.  `out[i]` receives the grid
// sum of v[i] (written by the last CTA only).
template <int NV>
__device__ __forceinline__ void grid_reduce_finish(double (&v)[NV], RedWs ws, double* out) {
  __shared__ double sred[kWarps][NV];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double s = warp_sum(v[i]);
    if (lane == 0) sred[warp][i] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sred[w][threadIdx.x];
    ws.partials[static_cast<int64_t>(blockIdx.x) * NV + threadIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ws.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  sum_partials_block(ws.partials, gridDim.x, NV, [&](int i, double t) { out[i] = t; });
  if (threadIdx.x == 0) *ws.ticket = 0u;
}

}  // namespace kls
