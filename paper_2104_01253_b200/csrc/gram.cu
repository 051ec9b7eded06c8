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
#include "reduce.cuh"

namespace {

using namespace kls;

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

template <int NX, int RP>
__global__ void __launch_bounds__(kThreads, 2) gram_kernel(GramParams p) {
  extern __shared__ double sacc[];  // [kWarps][ng * kG * NX]
  __shared__ double sx[kWarps][NX + 1];
  __shared__ bool s_last;
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

  // CTA reduction of the per-thread extras
#pragma unroll
  for (int t = 0; t < NX; ++t) {
    const double s = warp_sum(ex[t]);
    if (lane == 0) sx[warp][t] = s;
  }
  {
    const double s = warp_sum(xn);
    if (lane == 0) sx[warp][NX] = s;
  }
  __syncthreads();

  const int has_b = p.bext != nullptr ? 1 : 0;
  const int nq = p.k * NX;
  const int nv = nq + has_b * NX + (p.xnorm ? 1 : 0);
  double* part = p.partials + static_cast<int64_t>(blockIdx.x) * nv;
  for (int i = threadIdx.x; i < nq; i += kThreads) {
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

  // last CTA: fixed-order sum over CTAs (4 interleaved accumulators)
  const int nb = gridDim.x;
  for (int i = threadIdx.x; i < nv; i += kThreads) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int b = 0;
    for (; b + 4 <= nb; b += 4) {
      a0 += __ldcg(p.partials + static_cast<int64_t>(b) * nv + i);
      a1 += __ldcg(p.partials + static_cast<int64_t>(b + 1) * nv + i);
      a2 += __ldcg(p.partials + static_cast<int64_t>(b + 2) * nv + i);
      a3 += __ldcg(p.partials + static_cast<int64_t>(b + 3) * nv + i);
    }
    for (; b < nb; ++b) a0 += __ldcg(p.partials + static_cast<int64_t>(b) * nv + i);
    const double s = (a0 + a1) + (a2 + a3);
    int64_t dst;
    if (i < nq) {
      dst = static_cast<int64_t>(i % NX) * p.out_ld + p.col0 + i / NX;
    } else if (has_b && i < nq + NX) {
      dst = static_cast<int64_t>(i - nq) * p.out_ld + p.bext_row;
    } else {
      dst = static_cast<int64_t>(NX) * p.out_ld;
    }
    p.out[dst] = s;
  }
  if (threadIdx.x == 0) *p.ticket = 0u;
}

constexpr int kRP = 4;                   // row pairs per lane per chunk
constexpr int kPanel = 1024;             // max Q columns per launch
constexpr int kBlocksPerSm = 2;

template <int NX>
int launch_gram(GramParams p, size_t ws_bytes, cudaStream_t st) {
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
  gram_kernel<NX, kRP><<<grid, kThreads, smem, st>>>(p);
  return check_launch("gram_kernel");
}

}  // namespace

// Generic fused reduction: out = [Q(:, 0:k), bext]^T [x0 (, x1)]  (+ x_last^2).
// Output is column-major with (k + (bext != NULL)) rows and nx columns, then
// one slot for x_last . x_last when xnorm != 0.  Mirrors kernels.mv_trans_mv
// (kernels.py:44-60) for the block shapes the solvers use.
KLS_API int kls_mv_trans_mv(const double* Q, int64_t ldq, int64_t m, int32_t k,
                            const double* bext, const double* x0, const double* x1, int32_t nx,
                            int32_t xnorm, double* out, void* ws, size_t ws_bytes, void* stream) {
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
    const int rc = nx == 1 ? launch_gram<1>(p, pws, st) : launch_gram<2>(p, pws, st);
    if (rc) return rc;
    c0 += kp;
  } while (c0 < k);
  return KLS_OK;
}

// The DCGS2 Arnoldi step reduction (arnoldi.py:362-370 plus the guard norm of
// arnoldi.py:414): out[0:j+1] = [Q, w]^T w, out[j+1:2j+2] = [Q, w]^T aw,
// out[2j+2] = aw . aw.  2j+3 doubles, the payload of the one allreduce.
KLS_API int kls_gram_dcgs2(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                           const double* aw, double* out, void* ws, size_t ws_bytes,
                           void* stream) {
  return kls_mv_trans_mv(Q, ldq, m, j, w, w, aw, 2, 1, out, ws, ws_bytes, stream);
}

// Workspace bytes that cover any reduction launch with up to kmax basis
// columns on the current device.
KLS_API size_t kls_workspace_bytes(int64_t m, int32_t kmax) {
  (void)m;
  const int64_t grid = (int64_t)kBlocksPerSm * sm_count();
  const int64_t nv = 2 * (int64_t)std::min(kmax, kPanel) + 2 * 2 + 1 + 8;
  return kTicketBytes + (size_t)(grid * nv) * sizeof(double);
}
