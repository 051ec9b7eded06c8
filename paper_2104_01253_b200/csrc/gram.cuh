// Shared pieces of the K1 fused-reduction kernels (gram_tma.cu: the
// cp.async.bulk / mbarrier staged streaming kernel; gram.cu: the one-CTA-
// per-output kernel for small m).  Both reduce over the fixed segment tree
// of seg.cuh, so their results do not depend on the number of ranks.
#pragma once

#include "peer.cuh"
#include "seg.cuh"
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
  int64_t m;         // local rows
  int32_t xnorm;     // append x_last . x_last
  int32_t out_ld;
  int32_t col0;      // output row of this panel's first Q column
  int32_t bext_row;  // output row of bext
  seg::Plan P;       // segments and items (rank-count-independent tree)
  seg::Ws ws;
  seg::Dest d;       // out / exports / fused peer exchange
  // DCGS2 step fusion (single panel, bext == x0): after the final sums the
  // finishing CTA also runs the device scalar step on out (dcgs2_scalars_block)
  double* coef;
  double* gout;
  int32_t qr;
  // 1: the producer streams the first chunk's Q tiles before waiting for
  // the preceding kernel -- only for launches whose predecessor writes none
  // of Q (the step plan's K2 -> operator -> K1 chain: the operator writes
  // Aw' only, and K2's q_j was complete before the operator passed its own
  // griddepcontrol.wait, which precedes its trigger)
  int32_t qprefetch;
};

constexpr int kG = 4;  // Q columns reduced together

__host__ __device__ inline int gram_nv(const GramParams& p, int nx) {
  return p.k * nx + (p.bext != nullptr ? nx : 0) + (p.xnorm ? 1 : 0);
}

// output position of reduced value i (Q columns first, then bext, then
// the x_last . x_last slot)
template <int NX>
__device__ __forceinline__ int64_t gram_dst(const GramParams& p, int i) {
  const int nq = p.k * NX;
  if (i < nq) return static_cast<int64_t>(i % NX) * p.out_ld + p.col0 + i / NX;
  if (p.bext != nullptr && i < nq + NX) return static_cast<int64_t>(i - nq) * p.out_ld + p.bext_row;
  return static_cast<int64_t>(NX) * p.out_ld;
}

// Rows [wbase, wbase + 64 RP) of one warp through 128-bit loads, rows past
// m read as zero (the < 64-row tail of a segment).  Operands already
// offset to the segment's first row.
struct GramRows {
  const double* Q;
  int64_t ldq;
  int32_t k;
  const double* bext;
  const double* x0;
  const double* x1;
  int64_t m;
  int32_t xnorm;
};

template <int NX, int RP, bool CHECK>
__device__ __forceinline__ void gram_chunk(const GramRows& p, int64_t wbase, int lane,
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

template <int NX>
int launch_gram_tma(GramParams p, cudaStream_t st);
bool tma_eligible(const GramParams& p);
// virtual CTAs per segment of the staged kernel (seg.cuh): one per 8192
// rows (so a medium-m launch is one item per CTA), at most this many (49:
// the 3 segments of an 8-rank share keep 147 of 148 SMs busy)
constexpr int kTmaVirt = 49;

}  // namespace gram
}  // namespace kls
