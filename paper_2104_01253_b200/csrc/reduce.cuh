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
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b)
      s += __ldcg(ws.partials + static_cast<int64_t>(b) * NV + threadIdx.x);
    out[threadIdx.x] = s;
  }
  if (threadIdx.x == 0) *ws.ticket = 0u;
}

}  // namespace kls
