// Shared pieces of the K1 fused-reduction kernels (gram.cu: 128-bit LDG
// streaming; gram_tma.cu: cp.async.bulk / mbarrier staged).
#pragma once

#include "peer.cuh"
#include "reduce.cuh"
#include "step.cuh"

namespace kls {
namespace gram {

struct GramParams {
  const double* Q;   // first column of this panel
  int64_t ldq;
  int32_t k;         // Q columns in this panel
  const double* bext;  // extra left column (counted after Q) or nullptr
  const double* x0;
  const double* x1;
  int64_t m;
  int32_t xnorm;     // append x_last . x_last
  double* out;       // column-major (out_ld x NX), then the xnorm slot
  int32_t out_ld;
  int32_t col0;      // output row of this panel's first Q column
  int32_t bext_row;  // output row of bext
  double* partials;  // [gridDim.x][nv]
  unsigned int* ticket;
  // fused one-shot allreduce over NVLink peers (peers.world > 1): the last
  // CTA exchanges the CTA-summed vector with every rank and writes the
  // rank-ordered global sum to `out`
  peer::Peers peers;
  uint64_t epoch;
  int* err;
  // DCGS2 step fusion (single panel, bext == x0): after the final sums the
  // last CTA also runs the device scalar step on out (dcgs2_scalars_block)
  double* coef;
  double* gout;
  int32_t qr;
};

constexpr int kG = 4;  // Q columns reduced together

template <int NX, int RP, bool CHECK>
__device__ __forceinline__ void gram_chunk(const GramParams& p, int64_t wbase, int lane,
                                           double* wacc, double (&ex)[NX], double& xn) {
  constexpr int V = kG * NX;
  const double* xs[2] = {p.x0, p.x1};
  double2 xv[NX][RP];
#pragma unroll
  for (int t = 0; t < NX; ++t)
#pragma unroll
    for (int r = 0; r < RP; ++r) xv[t][r] = load_pair<CHECK>(xs[t], wbase + 64 * r + 2 * lane, p.m);

  if (p.bext != nullptr) {
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      // the DCGS2 call passes bext == x0 (the pending w): reuse the registers
      const double2 b = p.bext == p.x0 ? xv[0][r]
                                        : load_pair<CHECK>(p.bext, wbase + 64 * r + 2 * lane, p.m);
#pragma unroll
      for (int t = 0; t < NX; ++t) {
        ex[t] = fma(b.x, xv[t][r].x, ex[t]);
        ex[t] = fma(b.y, xv[t][r].y, ex[t]);
      }
    }
  }
  if (p.xnorm) {
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      xn = fma(xv[NX - 1][r].x, xv[NX - 1][r].x, xn);
      xn = fma(xv[NX - 1][r].y, xv[NX - 1][r].y, xn);
    }
  }

  const int ng = (p.k + kG - 1) / kG;
  for (int g = 0; g < ng; ++g) {
    double2 q[kG][RP];
#pragma unroll
    for (int cc = 0; cc < kG; ++cc) {
      const int c = g * kG + cc;
      if (c < p.k) {
        const double* col = p.Q + static_cast<int64_t>(c) * p.ldq;
#pragma unroll
        for (int r = 0; r < RP; ++r) q[cc][r] = load_pair<CHECK>(col, wbase + 64 * r + 2 * lane, p.m);
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) q[cc][r] = make_double2(0.0, 0.0);
      }
    }
    double acc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] = 0.0;
#pragma unroll
    for (int cc = 0; cc < kG; ++cc)
#pragma unroll
      for (int r = 0; r < RP; ++r)
#pragma unroll
        for (int t = 0; t < NX; ++t) {
          acc[cc * NX + t] = fma(q[cc][r].x, xv[t][r].x, acc[cc * NX + t]);
          acc[cc * NX + t] = fma(q[cc][r].y, xv[t][r].y, acc[cc * NX + t]);
        }
    const double s = warp_transpose_reduce<V>(acc, lane);
    if ((lane & (32 / V - 1)) == 0) wacc[g * V + warp_slot<V>(lane)] += s;
  }
}

// CTA reduction + last-CTA fixed-order grid sum.  Called by every thread
// of the CTA; threads of warps >= kWarps (a producer warp) contribute
// nothing but take part in the barriers.
template <int NX>
__device__ __forceinline__ void gram_epilogue(const GramParams& p, const double* sacc, int stride,
                                              double (&ex)[NX], double xn) {
  __shared__ double sx[kWarps][NX + 1];
  __shared__ bool s_last;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool consumer = warp < kWarps;
  // the streaming is done: a dependent update (PDL) may start staging its
  // Q tiles while the partial sums and the scalar step finish here
  pdl_trigger();
  // CTA reduction of the per-thread extras
#pragma unroll
  for (int t = 0; t < NX; ++t) {
    const double s = warp_sum(ex[t]);
    if (lane == 0 && consumer) sx[warp][t] = s;
  }
  {
    const double s = warp_sum(xn);
    if (lane == 0 && consumer) sx[warp][NX] = s;
  }
  __syncthreads();

  const int has_b = p.bext != nullptr ? 1 : 0;
  const int nq = p.k * NX;
  const int nv = nq + has_b * NX + (p.xnorm ? 1 : 0);
  double* part = p.partials + static_cast<int64_t>(blockIdx.x) * nv;
  for (int i = threadIdx.x; i < nq; i += blockDim.x) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sacc[w * stride + i];
    part[i] = s;
  }
  if (threadIdx.x < NX && has_b) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sx[w][threadIdx.x];
    part[nq + threadIdx.x] = s;
  }
  if (threadIdx.x == 0 && p.xnorm) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) s += sx[w][NX];
    part[nv - 1] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(p.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // last CTA: fixed-order sum over CTAs (sum_partials_block)
  const int nb = gridDim.x;
  const bool fused = p.peers.world > 1;
  double* mine = fused ? peer::slot(p.peers.buf[p.peers.rank], p.peers.cap, p.epoch) : nullptr;
  auto dst_of = [&](int i) -> int64_t {
    if (i < nq) return static_cast<int64_t>(i % NX) * p.out_ld + p.col0 + i / NX;
    if (has_b && i < nq + NX) return static_cast<int64_t>(i - nq) * p.out_ld + p.bext_row;
    return static_cast<int64_t>(NX) * p.out_ld;
  };
  sum_partials_block(p.partials, nb, nv, [&](int i, double s) {
    if (fused)
      mine[i] = s;
    else
      p.out[dst_of(i)] = s;
  });
  if (threadIdx.x == 0) *p.ticket = 0u;
  if (!fused) {
    if (p.coef != nullptr) {
      __syncthreads();
      dcgs2_scalars_block(p.out, p.bext_row, p.qr, p.coef, p.gout);
    }
    return;
  }
  // one-shot exchange: publish, signal every peer, wait for every peer, then
  // sum the N slots in rank order (identical bits on every rank)
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < p.peers.world) {
    __threadfence_system();
    peer::st_release_sys(peer::ar_flags(p.peers.buf[threadIdx.x]) + p.peers.rank, p.epoch);
    if (!peer::wait_flag(peer::ar_flags(p.peers.buf[p.peers.rank]) + threadIdx.x, p.epoch))
      atomicExch(&s_ok, 0);
  }
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0) *p.err = 1;
    for (int i = threadIdx.x; i < nv; i += blockDim.x)
      p.out[dst_of(i)] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < p.peers.world; ++r) {
      const volatile double* v = peer::slot(p.peers.buf[r], p.peers.cap, p.epoch);
      s += v[i];
    }
    p.out[dst_of(i)] = s;
  }
  if (p.coef != nullptr) {
    __syncthreads();
    dcgs2_scalars_block(p.out, p.bext_row, p.qr, p.coef, p.gout);
  }
}

template <int NX>
int launch_gram_tma(GramParams p, size_t ws_bytes, cudaStream_t st);
bool tma_eligible(const GramParams& p);

}  // namespace gram
}  // namespace kls
