// K1: fused block inner products  g = [Q, b]^T [x0, x1]  (+ x_last . x_last).
//
// Replaces the reference's single global reduction of a DCGS2 step,
//   left  = np.hstack([Q, w]);  right = np.column_stack([w, aw])
//   g     = mv_trans_mv(left, right)                 (arnoldi.py:362-366,
//                                                     kernels.py:44-60)
// without materialising the hstack copy, and folds in the uncounted guard
// norm ||aw|| of arnoldi.py:414.  One streaming pass over the j columns of Q
// plus the two vectors: 8 m (j + 2) bytes from HBM.
//
// Structure (DESIGN.md §4 K1): a persistent grid of 2 CTAs per SM walks row
// chunks; each warp owns 64*RP contiguous rows of a chunk, keeps its slice of
// x0/x1 in registers, streams G columns of Q at a time with 128-bit loads,
// and reduce-scatters the G*NX partial dots across the warp with a halving
// butterfly.  Per-warp accumulators live in shared memory; the CTA partials
// land in a workspace and the last CTA to finish (atomic ticket) sums them in
// fixed CTA order.  Every sum has a fixed order, so results are bitwise
// reproducible run to run (the reference's determinism rule, kernels.py:11-12).
#include "gram.cuh"

#include <cstdlib>

namespace {

using namespace kls;
using namespace kls::gram;

template <int NX, int RP>
__global__ void __launch_bounds__(kThreads, 2) gram_kernel(GramParams p) {
  pdl_wait();  // x vectors / basis from the preceding kernels
  extern __shared__ double sacc[];  // [kWarps][ng * kG * NX]
  constexpr int V = kG * NX;
  constexpr int64_t WROWS = 64 * RP;
  constexpr int64_t CROWS = WROWS * kWarps;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ng = (p.k + kG - 1) / kG;
  const int stride = ng * V;
  double* wacc = sacc + warp * stride;
  for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
  __syncwarp();

  double ex[NX];
#pragma unroll
  for (int t = 0; t < NX; ++t) ex[t] = 0.0;
  double xn = 0.0;

  const int64_t nchunks = (p.m + CROWS - 1) / CROWS;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t cbase = ch * CROWS;
    const int64_t wbase = cbase + warp * WROWS;
    if (cbase + CROWS <= p.m)
      gram_chunk<NX, RP, false>(p, wbase, lane, wacc, ex, xn);
    else
      gram_chunk<NX, RP, true>(p, wbase, lane, wacc, ex, xn);
  }

  gram_epilogue<NX>(p, sacc, stride, ex, xn);
}

// Small-m K1 (a few 1e4..1e5 local rows, where the chunked kernels leave
// most SMs idle and walk the columns as a serial chain): one 64-row block per
// CTA, the CTA's 8 warps splitting the column groups, so a 1e4-row Gram pass
// spreads over ~150 SMs and each warp issues its loads at once.  Same
// per-group butterfly and epilogue as gram_kernel.
template <int NX, bool CHECK>
__device__ __forceinline__ void gram_small_block(const GramParams& p, int64_t row, int warp,
                                                 int lane, double* wacc, double (&ex)[NX],
                                                 double& xn) {
  constexpr int V = kG * NX;
  const double* xs[2] = {p.x0, p.x1};
  double2 xv[NX];
#pragma unroll
  for (int t = 0; t < NX; ++t) xv[t] = load_pair<CHECK>(xs[t], row, p.m);
  if (warp == 0) {
    if (p.bext != nullptr) {
      const double2 b = p.bext == p.x0 ? xv[0] : load_pair<CHECK>(p.bext, row, p.m);
#pragma unroll
      for (int t = 0; t < NX; ++t) {
        ex[t] = fma(b.x, xv[t].x, ex[t]);
        ex[t] = fma(b.y, xv[t].y, ex[t]);
      }
    }
    if (p.xnorm) {
      xn = fma(xv[NX - 1].x, xv[NX - 1].x, xn);
      xn = fma(xv[NX - 1].y, xv[NX - 1].y, xn);
    }
  }
  const int ng = (p.k + kG - 1) / kG;
#pragma unroll 2
  for (int g = warp; g < ng; g += kWarps) {
    double2 q[kG];
#pragma unroll
    for (int cc = 0; cc < kG; ++cc) {
      const int c = g * kG + cc;
      q[cc] = c < p.k ? load_pair<CHECK>(p.Q + static_cast<int64_t>(c) * p.ldq, row, p.m)
                      : make_double2(0.0, 0.0);
    }
    double acc[V];
#pragma unroll
    for (int cc = 0; cc < kG; ++cc)
#pragma unroll
      for (int t = 0; t < NX; ++t) {
        acc[cc * NX + t] = fma(q[cc].x, xv[t].x, 0.0);
        acc[cc * NX + t] = fma(q[cc].y, xv[t].y, acc[cc * NX + t]);
      }
    const double sred = warp_transpose_reduce<V>(acc, lane);
    if ((lane & (32 / V - 1)) == 0) wacc[g * V + warp_slot<V>(lane)] += sred;
  }
}

template <int NX>
__global__ void __launch_bounds__(kThreads, 2) gram_small_kernel(GramParams p) {
  pdl_wait();
  extern __shared__ double sacc[];  // [kWarps][ng * kG * NX]
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int stride = (p.k + kG - 1) / kG * kG * NX;
  double* wacc = sacc + warp * stride;
  for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
  __syncwarp();
  double ex[NX];
#pragma unroll
  for (int t = 0; t < NX; ++t) ex[t] = 0.0;
  double xn = 0.0;
  const int64_t nblk = (p.m + 63) / 64;
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int64_t row = b * 64 + 2 * lane;
    if (b * 64 + 64 <= p.m)
      gram_small_block<NX, false>(p, row, warp, lane, wacc, ex, xn);
    else
      gram_small_block<NX, true>(p, row, warp, lane, wacc, ex, xn);
  }
  gram_epilogue<NX>(p, sacc, stride, ex, xn);
}

// Latency-bound K1 for the smallest m (config 1, the GMRES / Krylov-Schur
// tails on one GPU): one CTA per output row — CTA c forms row c of
// [Q, bext]^T [x0 (, x1)] (or the x_last . x_last slot) over all m rows — so
// no CTA ever waits on another's partial sums: each output is one CTA's
// fixed-order tree (4 strided row-pair accumulators per thread, warp
// butterflies, warps in index order).  The last CTA to finish (ticket) runs
// the fused DCGS2 scalar step on the staged result.  At m = 1e4 the chunked
// small kernel spent most of its time in the cross-CTA partial sum.
constexpr int kColThreads = 512;
constexpr int64_t kColRows = 1 << 14;  // at or below this m (one GPU) gram_cols_kernel is used

template <int NX>
__global__ void __launch_bounds__(kColThreads) gram_cols_kernel(GramParams p) {
  extern __shared__ double sg[];  // staged g (2k + 3) for the scalar step
  __shared__ double sred[kColThreads / 32][NX];
  __shared__ bool s_last;
  pdl_wait();
  const int c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool has_b = p.bext != nullptr;
  const bool norm_row = c >= p.k + (has_b ? 1 : 0);  // the x_last . x_last slot
  const double* left = c < p.k ? p.Q + static_cast<int64_t>(c) * p.ldq
                       : has_b && c == p.k ? p.bext
                                           : (NX == 2 ? p.x1 : p.x0);
  const double* xs[2] = {norm_row ? left : p.x0, norm_row ? left : p.x1};
  constexpr int U = 4;
  double acc[NX][U];
#pragma unroll
  for (int t = 0; t < NX; ++t)
#pragma unroll
    for (int u = 0; u < U; ++u) acc[t][u] = 0.0;
  const int nt = norm_row ? 1 : NX;
  const int64_t npair = p.m / 2;
  const double2* l2 = reinterpret_cast<const double2*>(left);
  int64_t i = tid;
  for (; i + (U - 1) * kColThreads < npair; i += U * kColThreads) {
    double2 a[U], x[NX][U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = l2[i + u * kColThreads];
#pragma unroll
    for (int t = 0; t < NX; ++t)
      if (t < nt)
#pragma unroll
        for (int u = 0; u < U; ++u)
          x[t][u] = reinterpret_cast<const double2*>(xs[t])[i + u * kColThreads];
#pragma unroll
    for (int t = 0; t < NX; ++t)
      if (t < nt)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          acc[t][u] = fma(a[u].x, x[t][u].x, acc[t][u]);
          acc[t][u] = fma(a[u].y, x[t][u].y, acc[t][u]);
        }
  }
  for (; i < npair; i += kColThreads) {
    const double2 a = l2[i];
#pragma unroll
    for (int t = 0; t < NX; ++t)
      if (t < nt) {
        const double2 x = reinterpret_cast<const double2*>(xs[t])[i];
        acc[t][0] = fma(a.x, x.x, acc[t][0]);
        acc[t][0] = fma(a.y, x.y, acc[t][0]);
      }
  }
  if ((p.m & 1) && tid == 0) {
#pragma unroll
    for (int t = 0; t < NX; ++t)
      if (t < nt) acc[t][0] = fma(left[p.m - 1], xs[t][p.m - 1], acc[t][0]);
  }
#pragma unroll
  for (int t = 0; t < NX; ++t) {
    const double v = warp_sum((acc[t][0] + acc[t][1]) + (acc[t][2] + acc[t][3]));
    if (lane == 0) sred[warp][t] = v;
  }
  __syncthreads();
  if (tid < nt) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kColThreads / 32; ++w) v += sred[w][tid];
    const int64_t dst = norm_row ? static_cast<int64_t>(NX) * p.out_ld
                        : c < p.k ? static_cast<int64_t>(tid) * p.out_ld + p.col0 + c
                                  : static_cast<int64_t>(tid) * p.out_ld + p.bext_row;
    p.out[dst] = v;
  }
  pdl_trigger();
  if (p.coef == nullptr) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(p.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int ng = 2 * p.bext_row + 3;
  for (int k = tid; k < ng; k += kColThreads) sg[k] = __ldcg(p.out + k);
  __syncthreads();
  dcgs2_scalars_block(sg, p.bext_row, p.qr, p.coef, p.gout);
  if (tid == 0) *p.ticket = 0u;
}

template <int NX>
int launch_gram_cols(GramParams p, cudaStream_t st) {
  const int grid = p.k + (p.bext != nullptr ? 1 : 0) + (p.xnorm ? 1 : 0);
  if (grid == 0) return KLS_OK;  // nothing to reduce (and no scalar step: it needs bext)
  const size_t smem = p.coef != nullptr ? sizeof(double) * (2 * static_cast<size_t>(p.bext_row) + 3) : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(gram_cols_kernel<NX>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "gram_cols: smem attr: %s", cudaGetErrorString(e));
  }
  return launch_dependent(gram_cols_kernel<NX>, dim3(grid), dim3(kColThreads), smem, st,
                          "gram_cols_kernel", p);
}

constexpr int64_t kSmallRows = 1 << 15;  // at or below this the small-m K1 is used (scripts/small_probe.py)
constexpr int kRP = 4;                   // row pairs per lane per chunk
constexpr int kPanel = 1024;             // max Q columns per launch
constexpr int kBlocksPerSm = 2;

// K1 variant: 1 = cp.async.bulk staged (gram_tma.cu, the default: 7.3 TB/s
// vs 7.1 TB/s for LDG at m = 1.3e8, j = 50..100), 0 = 128-bit LDG streaming,
// 2 = never the small-m kernel.  KLS_GRAM=ldg|tma|big overrides it for
// experiments.
int gram_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KLS_GRAM");
    v = (e && e[0] == 'l') ? 0 : (e && e[0] == 'b') ? 2 : 1;
  }
  return v;
}

template <int NX>
int launch_gram_small(GramParams p, size_t ws_bytes, cudaStream_t st) {
  // ~4 row blocks per CTA: enough CTAs to spread the rows, few enough that
  // the last CTA's sum over the partials stays short
  const int64_t nblk = ceil_div(p.m, 64);
  int grid = static_cast<int>(std::min<int64_t>(std::max<int64_t>(ceil_div(nblk, 4), 32),
                                                (int64_t)kBlocksPerSm * sm_count()));
  grid = static_cast<int>(std::min<int64_t>(grid, nblk));
  if (grid < 1) grid = 1;
  const int has_b = p.bext != nullptr ? 1 : 0;
  const int64_t nv = (int64_t)p.k * NX + has_b * NX + (p.xnorm ? 1 : 0);
  if (!red_ws_fits(ws_bytes, grid, static_cast<int>(nv)))
    return fail(KLS_ENOSPC, "gram_small: workspace too small");
  const size_t smem = (size_t)kWarps * ((p.k + kG - 1) / kG) * kG * NX * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(gram_small_kernel<NX>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "gram_small: smem attr: %s", cudaGetErrorString(e));
  }
  return launch_dependent(gram_small_kernel<NX>, dim3(grid), dim3(kThreads), smem, st,
                          "gram_small_kernel", p);
}

template <int NX>
int launch_gram(GramParams p, size_t ws_bytes, cudaStream_t st) {
  if (p.m <= kColRows && p.m >= 2 && p.peers.world <= 1 && gram_variant() == 1)
    return launch_gram_cols<NX>(p, st);
  if (p.m <= kSmallRows && p.k > 0 && p.k <= kPanel && gram_variant() != 2)
    return launch_gram_small<NX>(p, ws_bytes, st);
  if (gram_variant() != 0 && tma_eligible(p)) return launch_gram_tma<NX>(p, ws_bytes, st);
  constexpr int64_t CROWS = 64 * kRP * kWarps;
  const int64_t nchunks = ceil_div(p.m, CROWS);
  int grid = static_cast<int>(std::min<int64_t>(nchunks, (int64_t)kBlocksPerSm * sm_count()));
  if (grid < 1) grid = 1;
  const int has_b = p.bext != nullptr ? 1 : 0;
  const int64_t nv = (int64_t)p.k * NX + has_b * NX + (p.xnorm ? 1 : 0);
  if (kTicketBytes + (size_t)grid * nv * sizeof(double) > ws_bytes)
    return fail(KLS_ENOSPC, "gram: workspace %zu bytes < %zu needed", ws_bytes,
                kTicketBytes + (size_t)grid * nv * sizeof(double));
  const int ng = (p.k + kG - 1) / kG;
  const size_t smem = (size_t)kWarps * ng * kG * NX * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(gram_kernel<NX, kRP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "gram: smem attr: %s", cudaGetErrorString(e));
  }
  return launch_dependent(gram_kernel<NX, kRP>, dim3(grid), dim3(kThreads), smem, st,
                          "gram_kernel", p);
}

}  // namespace

// Generic fused reduction: out = [Q(:, 0:k), bext]^T [x0 (, x1)]  (+ x_last^2).
// Output is column-major with (k + (bext != NULL)) rows and nx columns, then
// one slot for x_last . x_last when xnorm != 0.  Mirrors kernels.mv_trans_mv
// (kernels.py:44-60) for the block shapes the solvers use.
static int mv_trans_mv_impl(const double* Q, int64_t ldq, int64_t m, int32_t k,
                            const double* bext, const double* x0, const double* x1, int32_t nx,
                            int32_t xnorm, double* out, void* ws, size_t ws_bytes, void* stream,
                            const peer::Peers* peers, uint64_t epoch, int* err,
                            double* coef = nullptr, double* gout = nullptr, int32_t qr = 0) {
  if (m < 0 || k < 0 || (k > 0 && (Q == nullptr || ldq < m)) || x0 == nullptr || out == nullptr ||
      ws == nullptr || (nx != 1 && nx != 2) || (nx == 2 && x1 == nullptr))
    return fail(KLS_EINVAL, "mv_trans_mv: bad arguments (m=%lld k=%d nx=%d)", (long long)m, k, nx);
  if ((reinterpret_cast<uintptr_t>(x0) | reinterpret_cast<uintptr_t>(x1) |
       reinterpret_cast<uintptr_t>(bext) | reinterpret_cast<uintptr_t>(Q)) & 15)
    return fail(KLS_EINVAL, "mv_trans_mv: operands must be 16-byte aligned");
  if (k > 0 && (ldq & 1)) return fail(KLS_EINVAL, "mv_trans_mv: ldq must be even");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int out_ld = k + (bext ? 1 : 0);
  unsigned int* ticket = static_cast<unsigned int*>(ws);
  double* partials = reinterpret_cast<double*>(static_cast<char*>(ws) + kTicketBytes);
  const size_t pws = ws_bytes;
  if (peers != nullptr && k > kPanel)
    return fail(KLS_EINVAL, "mv_trans_mv: the fused peer exchange needs k <= %d", kPanel);
  if (coef != nullptr && k > kPanel)
    return fail(KLS_EINVAL, "gram_dcgs2_step: the fused scalar step needs j <= %d", kPanel);
  // panels of <= kPanel columns; extras ride on the last panel
  int c0 = 0;
  do {
    const int kp = std::min(kPanel, k - c0);
    const bool last = c0 + kp >= k;
    GramParams p;
    p.Q = Q ? Q + (int64_t)c0 * ldq : nullptr;
    p.ldq = ldq;
    p.k = kp;
    p.bext = last ? bext : nullptr;
    p.x0 = x0;
    p.x1 = nx == 2 ? x1 : nullptr;
    p.m = m;
    p.xnorm = last ? xnorm : 0;
    p.out = out;
    p.out_ld = out_ld;
    p.col0 = c0;
    p.bext_row = k;
    p.partials = partials;
    p.ticket = ticket;
    p.peers.world = 0;
    p.epoch = epoch;
    p.err = err;
    p.coef = last ? coef : nullptr;
    p.gout = gout;
    p.qr = qr;
    if (peers != nullptr) p.peers = *peers;
    const int rc = nx == 1 ? launch_gram<1>(p, pws, st) : launch_gram<2>(p, pws, st);
    if (rc) return rc;
    c0 += kp;
  } while (c0 < k);
  return KLS_OK;
}

KLS_API int kls_mv_trans_mv(const double* Q, int64_t ldq, int64_t m, int32_t k,
                            const double* bext, const double* x0, const double* x1, int32_t nx,
                            int32_t xnorm, double* out, void* ws, size_t ws_bytes, void* stream) {
  return mv_trans_mv_impl(Q, ldq, m, k, bext, x0, x1, nx, xnorm, out, ws, ws_bytes, stream,
                          nullptr, 0, nullptr);
}

// The DCGS2 Arnoldi step reduction (arnoldi.py:362-370 plus the guard norm of
// arnoldi.py:414): out[0:j+1] = [Q, w]^T w, out[j+1:2j+2] = [Q, w]^T aw,
// out[2j+2] = aw . aw.  2j+3 doubles, the payload of the one allreduce.
KLS_API int kls_gram_dcgs2(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                           const double* aw, double* out, void* ws, size_t ws_bytes,
                           void* stream) {
  return kls_mv_trans_mv(Q, ldq, m, j, w, w, aw, 2, 1, out, ws, ws_bytes, stream);
}

// kls_gram_dcgs2 fused with the step's global reduction: the kernel's last
// CTA exchanges the local 2j+3 sums with every rank over NVLink peer memory
// (symmetric buffers bufs[0..world), as kls_peer_allreduce) and writes the
// rank-ordered global sum to out — compute and collective in one launch.
KLS_API int kls_gram_dcgs2_peer(const double* Q, int64_t ldq, int64_t m, int32_t j,
                                const double* w, const double* aw, double* out, void* ws,
                                size_t ws_bytes, void* const* bufs, int32_t rank, int32_t world,
                                int32_t cap, uint64_t epoch, int* err, void* stream) {
  if (bufs == nullptr || err == nullptr || world < 2 || world > peer::kMaxPeers || rank < 0 ||
      rank >= world || 2 * j + 3 > cap)
    return fail(KLS_EINVAL, "gram_dcgs2_peer: bad peer arguments");
  peer::Peers pr;
  for (int r = 0; r < peer::kMaxPeers; ++r) pr.buf[r] = r < world ? static_cast<char*>(bufs[r]) : nullptr;
  pr.rank = rank;
  pr.world = world;
  pr.cap = cap;
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, ws, ws_bytes, stream, &pr, epoch,
                          err);
}

// kls_gram_dcgs2 with the step's device scalar arithmetic fused into the
// kernel's last CTA (kls_dcgs2_scalars): g -> out (device), the update
// coefficients [c, s/alpha (QR: s), t_piv, alpha] -> coef, and g -> gout
// (mapped host memory, may be NULL).  One launch per step instead of two.
KLS_API int kls_gram_dcgs2_step(const double* Q, int64_t ldq, int64_t m, int32_t j,
                                const double* w, const double* aw, double* out, double* coef,
                                double* gout, int32_t qr, void* ws, size_t ws_bytes, void* stream) {
  if (coef == nullptr) return fail(KLS_EINVAL, "gram_dcgs2_step: null coefficient buffer");
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, ws, ws_bytes, stream, nullptr, 0,
                          nullptr, coef, gout, qr);
}

// The same fused with the peer allreduce (kls_gram_dcgs2_peer): Gram pass,
// global reduction and scalar step in one launch.
KLS_API int kls_gram_dcgs2_peer_step(const double* Q, int64_t ldq, int64_t m, int32_t j,
                                     const double* w, const double* aw, double* out, double* coef,
                                     double* gout, int32_t qr, void* ws, size_t ws_bytes,
                                     void* const* bufs, int32_t rank, int32_t world, int32_t cap,
                                     uint64_t epoch, int* err, void* stream) {
  if (coef == nullptr || bufs == nullptr || err == nullptr || world < 2 ||
      world > peer::kMaxPeers || rank < 0 || rank >= world || 2 * j + 3 > cap)
    return fail(KLS_EINVAL, "gram_dcgs2_peer_step: bad arguments");
  peer::Peers pr;
  for (int r = 0; r < peer::kMaxPeers; ++r) pr.buf[r] = r < world ? static_cast<char*>(bufs[r]) : nullptr;
  pr.rank = rank;
  pr.world = world;
  pr.cap = cap;
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, ws, ws_bytes, stream, &pr, epoch,
                          err, coef, gout, qr);
}

// Workspace bytes that cover any reduction launch with up to kmax basis
// columns on the current device.
KLS_API size_t kls_workspace_bytes(int64_t m, int32_t kmax) {
  (void)m;
  const int64_t grid = (int64_t)kBlocksPerSm * sm_count();
  const int64_t nv = 2 * (int64_t)std::min(kmax, kPanel) + 2 * 2 + 1 + 8;
  return kTicketBytes + (size_t)(grid * nv) * sizeof(double);
}
