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
// Two kernels, chosen by the GLOBAL row count (so every rank of a sharded
// run uses the same one): the TMA-staged persistent kernel (gram_tma.cu)
// and, for m <= 32 K rows (config 1, the GMRES / Krylov-Schur tails), one
// CTA per output row.  Both sum over the fixed segment tree of seg.cuh:
// the result does not depend on the number of ranks (or on the physical
// grid), and repeated runs are bitwise identical (the reference's
// determinism rule, kernels.py:11-12).
#include "gram.cuh"

#include <cstdlib>

namespace {

using namespace kls;
using namespace kls::gram;

// One CTA per output row: CTA c forms row c of [Q, bext]^T [x0 (, x1)] (or
// the x_last . x_last slot) over the rank's rows.  Warp w reduces the local
// segments w, w + 16, ...: lane l takes the segment's row pairs l, l + 32,
// ... (an fma chain), then a warp butterfly -- the segment value.  The
// CTA evaluates its output's local segment tree; with several ranks it
// publishes the exported nodes, and the last CTA to finish (ticket)
// exchanges them (fused peers) and runs the fused DCGS2 scalar step.
constexpr int kColThreads = 768;  // 24 warps: one per local segment
constexpr int kColWarps = kColThreads / 32;
constexpr int64_t kColRows = 1 << 15;  // global m at or below this: gram_cols_kernel

template <int NX>
__global__ void __launch_bounds__(kColThreads) gram_cols_kernel(GramParams p) {
  extern __shared__ double sg[];  // staged g (2k + 3) for the scalar step
  __shared__ double s_seg[seg::kG][NX];
  __shared__ int s_last, s_ok;
  pdl_wait();
  const int c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool has_b = p.bext != nullptr;
  const bool norm_row = c >= p.k + (has_b ? 1 : 0);  // the x_last . x_last slot
  const double* left = c < p.k ? p.Q + static_cast<int64_t>(c) * p.ldq
                       : has_b && c == p.k ? p.bext
                                           : (NX == 2 ? p.x1 : p.x0);
  const double* xs[2] = {norm_row ? left : p.x0, norm_row ? left : p.x1};
  const int nt = norm_row ? 1 : NX;
  const int nq = p.k * NX;
  const int nv = gram_nv(p, NX);
  for (int s = warp; s < p.P.L.nseg; s += kColWarps) {
    const int64_t a = p.P.L.off[s];  // even (segment boundaries)
    const int64_t rows = p.P.L.off[s + 1] - a;
    double acc[NX];
#pragma unroll
    for (int t = 0; t < NX; ++t) acc[t] = 0.0;
    const double2* l2 = reinterpret_cast<const double2*>(left + a);
    const double2* x2[2] = {reinterpret_cast<const double2*>(xs[0] + a),
                            reinterpret_cast<const double2*>(xs[NX - 1] + a)};
    const int64_t npair = rows / 2;
    int64_t i = lane;
    // four row pairs' loads in flight, then their fmas in row order (the
    // same sequential per-lane chain as the one-pair loop below)
    for (; i + 96 < npair; i += 128) {
      double2 av[4], xv[NX][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        av[u] = l2[i + 32 * u];
#pragma unroll
        for (int t = 0; t < NX; ++t)
          if (t < nt) xv[t][u] = x2[t][i + 32 * u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int t = 0; t < NX; ++t)
          if (t < nt) {
            acc[t] = fma(av[u].x, xv[t][u].x, acc[t]);
            acc[t] = fma(av[u].y, xv[t][u].y, acc[t]);
          }
    }
    for (; i < npair; i += 32) {
      const double2 av = l2[i];
#pragma unroll
      for (int t = 0; t < NX; ++t)
        if (t < nt) {
          const double2 x = x2[t][i];
          acc[t] = fma(av.x, x.x, acc[t]);
          acc[t] = fma(av.y, x.y, acc[t]);
        }
    }
    if ((rows & 1) && lane == 0) {
#pragma unroll
      for (int t = 0; t < NX; ++t)
        if (t < nt) acc[t] = fma(left[a + rows - 1], xs[t][a + rows - 1], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < NX; ++t) {
      const double v = warp_sum(acc[t]);
      if (lane == 0) s_seg[s][t] = v;
    }
  }
  __syncthreads();
  const seg::Layout& L = p.P.L;
  const bool fused = L.world > 1 && p.d.peers.world > 1;
  if (tid < nt) {
    const int i = norm_row ? nv - 1 : c < p.k ? c * NX + tid : nq + tid;
    const int64_t dst = gram_dst<NX>(p, i);
    if (L.world == 1) {
      p.d.out[dst] = seg::root24([&](int s) { return s_seg[s][tid]; });
    } else {
      double val[seg::kNodes];
      seg::local_tree_from(L, [&](int s) { return s_seg[s][tid]; }, val);
      int ids[seg::kMaxExport];
      const int ne = seg::exports(L.gseg0, L.gseg0 + L.nseg, ids);
      double* mine = fused ? peer::slot(p.d.peers.buf[p.d.peers.rank], p.d.peers.cap, p.d.epoch) : nullptr;
      for (int e = 0; e < ne; ++e) {
        if (fused)
          mine[static_cast<int64_t>(e) * nv + i] = val[ids[e]];
        else
          p.d.out[static_cast<int64_t>(e) * p.d.xstride + dst] = val[ids[e]];
      }
    }
  }
  pdl_trigger();
  if (!fused && p.coef == nullptr) return;
  if (fused)
    __threadfence_system();  // the exports in this rank's peer slot, before the exchange
  else
    __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(p.ws.tick + seg::kG, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) p.ws.tick[seg::kG] = 0u;
  if (fused) {
    if (!seg::peer_exchange<kColThreads, 0>(p.d, tid, &s_ok)) {
      if (tid == 0) *p.d.err = 1;
      for (int i = tid; i < nv; i += kColThreads)
        p.d.out[gram_dst<NX>(p, i)] = __longlong_as_double(0x7ff8000000000000ll);
      return;
    }
    seg::combine_from_slots<kColThreads>(p.d, nv, tid,
                                         [&](int i, double v) { p.d.out[gram_dst<NX>(p, i)] = v; });
    __threadfence();
    __syncthreads();
  }
  if (p.coef == nullptr) return;
  const int ng = 2 * p.bext_row + 3;
  for (int k = tid; k < ng; k += kColThreads) sg[k] = __ldcg(p.d.out + k);
  __syncthreads();
  dcgs2_scalars_block(sg, p.bext_row, p.qr, p.coef, p.gout);
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

constexpr int kPanel = 256;  // max Q columns per launch

template <int NX>
int launch_gram(GramParams p, int64_t m_global, size_t ws_bytes, cudaStream_t st) {
  if (m_global <= kColRows) {
    if (ws_bytes < seg::kTickBytes) return fail(KLS_ENOSPC, "gram: workspace too small");
    return launch_gram_cols<NX>(p, st);
  }
  if (!tma_eligible(p)) return fail(KLS_EINVAL, "gram: operands must be 16-byte aligned, ldq even");
  static const int vmax = [] {  // KLS_TMA_VIRT: experiments only (changes the tree)
    const char* e = getenv("KLS_TMA_VIRT");
    return e != nullptr && atoi(e) > 0 ? atoi(e) : kTmaVirt;
  }();
  seg::make_plan(p.P.L, 8192, vmax, p.P);
  const int nv = gram_nv(p, NX);
  if (seg::plan_ws_bytes(p.P, nv) > ws_bytes)
    return fail(KLS_ENOSPC, "gram: workspace %zu bytes < %zu needed", ws_bytes,
                seg::plan_ws_bytes(p.P, nv));
  p.ws = seg::ws_of(p.ws.tick, p.P.nitems, nv);
  return launch_gram_tma<NX>(p, st);
}

}  // namespace

// Generic fused reduction: out = [Q(:, 0:k), bext]^T [x0 (, x1)]  (+ x_last^2).
// Output is column-major with (k + (bext != NULL)) rows and nx columns, then
// one slot for x_last . x_last when xnorm != 0.  Mirrors kernels.mv_trans_mv
// (kernels.py:44-60) for the block shapes the solvers use.
static int mv_trans_mv_impl(const double* Q, int64_t ldq, int64_t m, int32_t k,
                            const double* bext, const double* x0, const double* x1, int32_t nx,
                            int32_t xnorm, double* out, const KlsSegs* segs, void* ws,
                            size_t ws_bytes, void* stream, const peer::Peers* peers,
                            uint64_t epoch, int* err, double* coef = nullptr,
                            double* gout = nullptr, int32_t qr = 0, int32_t qprefetch = 0) {
  // a rank may hold no rows (m = 0: empty tensors, null pointers); it still
  // takes part in the reduction tree and the exchange
  if (m < 0 || k < 0 || (k > 0 && ((m > 0 && Q == nullptr) || ldq < m)) ||
      (m > 0 && x0 == nullptr) || out == nullptr || ws == nullptr || (nx != 1 && nx != 2) ||
      (nx == 2 && m > 0 && x1 == nullptr))
    return fail(KLS_EINVAL, "mv_trans_mv: bad arguments (m=%lld k=%d nx=%d)", (long long)m, k, nx);
  if ((reinterpret_cast<uintptr_t>(x0) | reinterpret_cast<uintptr_t>(x1) |
       reinterpret_cast<uintptr_t>(bext) | reinterpret_cast<uintptr_t>(Q)) & 15)
    return fail(KLS_EINVAL, "mv_trans_mv: operands must be 16-byte aligned");
  if (k > 0 && (ldq & 1)) return fail(KLS_EINVAL, "mv_trans_mv: ldq must be even");
  seg::Layout L;
  int rc = seg::make_layout(segs, m, L);
  if (rc) return rc;
  const int64_t m_global = segs != nullptr ? segs->m : m;
  if (peers != nullptr && (peers->world != L.world || peers->rank != L.rank))
    return fail(KLS_EINVAL, "mv_trans_mv: peer table (rank %d of %d) does not match the layout "
                "(rank %d of %d)", peers->rank, peers->world, L.rank, L.world);
  if (coef != nullptr && L.world > 1 && peers == nullptr)
    return fail(KLS_EINVAL, "gram_dcgs2_step: with several ranks the scalar step needs the "
                "fused peer exchange");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int out_ld = k + (bext ? 1 : 0);
  // panels of <= kPanel columns; extras (and the scalar step) ride on the
  // last panel; with a fused peer exchange panel i uses epoch + i
  int c0 = 0;
  uint64_t panel = 0;
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
    p.out_ld = out_ld;
    p.col0 = c0;
    p.bext_row = k;
    p.P.L = L;
    p.P.nitems = 0;
    p.ws = seg::ws_of(ws, 0, 0);
    p.d.out = out;
    p.d.xstride = static_cast<int64_t>(out_ld) * nx + (xnorm ? 1 : 0);
    p.d.peers.world = 0;
    p.d.epoch = epoch + panel++;
    p.d.err = err;
    p.coef = last ? coef : nullptr;
    p.gout = gout;
    p.qr = qr;
    p.qprefetch = qprefetch;
    if (peers != nullptr) p.d.peers = *peers;
    if (peers != nullptr && seg::kMaxExport * gram_nv(p, nx) > peers->cap)
      return fail(KLS_EINVAL, "mv_trans_mv: %d exported values exceed the peer slot (%d)",
                  seg::kMaxExport * gram_nv(p, nx), peers->cap);
    rc = nx == 1 ? launch_gram<1>(p, m_global, ws_bytes, st)
                 : launch_gram<2>(p, m_global, ws_bytes, st);
    if (rc) return rc;
    c0 += kp;
  } while (c0 < k);
  return KLS_OK;
}

KLS_API int kls_mv_trans_mv(const double* Q, int64_t ldq, int64_t m, int32_t k,
                            const double* bext, const double* x0, const double* x1, int32_t nx,
                            int32_t xnorm, double* out, const KlsSegs* segs, void* ws,
                            size_t ws_bytes, void* stream) {
  return mv_trans_mv_impl(Q, ldq, m, k, bext, x0, x1, nx, xnorm, out, segs, ws, ws_bytes, stream,
                          nullptr, 0, nullptr);
}

// The DCGS2 Arnoldi step reduction (arnoldi.py:362-370 plus the guard norm of
// arnoldi.py:414): out[0:j+1] = [Q, w]^T w, out[j+1:2j+2] = [Q, w]^T aw,
// out[2j+2] = aw . aw.  2j+3 doubles, the payload of the one allreduce.
KLS_API int kls_gram_dcgs2(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                           const double* aw, double* out, const KlsSegs* segs, void* ws,
                           size_t ws_bytes, void* stream) {
  return kls_mv_trans_mv(Q, ldq, m, j, w, w, aw, 2, 1, out, segs, ws, ws_bytes, stream);
}

static int make_peer_table(peer::Peers& pr, void* const* bufs, int32_t rank, int32_t world,
                           int32_t cap) {
  if (bufs == nullptr || world < 2 || world > peer::kMaxPeers || rank < 0 || rank >= world ||
      cap < 1)
    return fail(KLS_EINVAL, "gram_dcgs2_peer: bad peer arguments");
  for (int r = 0; r < peer::kMaxPeers; ++r) pr.buf[r] = r < world ? static_cast<char*>(bufs[r]) : nullptr;
  pr.rank = rank;
  pr.world = world;
  pr.cap = cap;
  return KLS_OK;
}

// kls_gram_dcgs2 fused with the step's global reduction: the finishing CTA
// publishes this rank's exported tree nodes over NVLink peer memory
// (symmetric buffers bufs[0..world)) and evaluates the fixed segment tree
// -- compute and collective in one launch, the same bits on every rank and
// as on one GPU.  j > 256 runs as ceil(j / 256) column panels, panel i
// exchanging with epoch + i.
KLS_API int kls_gram_dcgs2_peer(const double* Q, int64_t ldq, int64_t m, int32_t j,
                                const double* w, const double* aw, double* out,
                                const KlsSegs* segs, void* ws, size_t ws_bytes, void* const* bufs,
                                int32_t rank, int32_t world, int32_t cap, uint64_t epoch,
                                int* err, void* stream) {
  peer::Peers pr;
  int rc = make_peer_table(pr, bufs, rank, world, cap);
  if (rc) return rc;
  if (err == nullptr) return fail(KLS_EINVAL, "gram_dcgs2_peer: null error flag");
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, segs, ws, ws_bytes, stream, &pr,
                          epoch, err);
}

// kls_gram_dcgs2 with the step's device scalar arithmetic fused into the
// finishing CTA (kls_dcgs2_scalars): g -> out (device), the update
// coefficients [c, s/alpha (QR: s), t_piv, alpha] -> coef, and g -> gout
// (mapped host memory, may be NULL).  One launch per step instead of two.
KLS_API int kls_gram_dcgs2_step(const double* Q, int64_t ldq, int64_t m, int32_t j,
                                const double* w, const double* aw, double* out, double* coef,
                                double* gout, int32_t qr, const KlsSegs* segs, void* ws,
                                size_t ws_bytes, void* stream) {
  if (coef == nullptr) return fail(KLS_EINVAL, "gram_dcgs2_step: null coefficient buffer");
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, segs, ws, ws_bytes, stream, nullptr,
                          0, nullptr, coef, gout, qr);
}

namespace kls {
// kls_gram_dcgs2_step for the step plan's K2 -> operator -> K1 chain
// (plan.cu): the Gram kernel streams its first chunk's Q tiles before
// waiting for the operator (GramParams::qprefetch).
int gram_dcgs2_step_chain(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                          const double* aw, double* out, double* coef, double* gout, int32_t qr,
                          const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream) {
  if (coef == nullptr) return fail(KLS_EINVAL, "gram_dcgs2_step: null coefficient buffer");
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, segs, ws, ws_bytes, stream, nullptr,
                          0, nullptr, coef, gout, qr, 1);
}
}  // namespace kls

// The same fused with the peer exchange (kls_gram_dcgs2_peer): Gram pass,
// global reduction and scalar step in one launch.
KLS_API int kls_gram_dcgs2_peer_step(const double* Q, int64_t ldq, int64_t m, int32_t j,
                                     const double* w, const double* aw, double* out, double* coef,
                                     double* gout, int32_t qr, const KlsSegs* segs, void* ws,
                                     size_t ws_bytes, void* const* bufs, int32_t rank,
                                     int32_t world, int32_t cap, uint64_t epoch, int* err,
                                     void* stream) {
  if (coef == nullptr || err == nullptr) return fail(KLS_EINVAL, "gram_dcgs2_peer_step: bad arguments");
  peer::Peers pr;
  int rc = make_peer_table(pr, bufs, rank, world, cap);
  if (rc) return rc;
  return mv_trans_mv_impl(Q, ldq, m, j, w, w, aw, 2, 1, out, segs, ws, ws_bytes, stream, &pr,
                          epoch, err, coef, gout, qr);
}

// Workspace bytes that cover any reduction launch with up to kmax basis
// columns: tickets, the item partials of the largest item plan (24
// segments x the largest virtual grid of any segmented kernel) and the 24
// segment values, for the widest reduction (a Gram panel, or CGS2's
// k + 1 outputs).
KLS_API size_t kls_workspace_bytes(int64_t m, int32_t kmax) {
  (void)m;
  const int64_t panel = std::min<int64_t>(kmax, kPanel);
  const int64_t nv = std::max<int64_t>(2 * panel + 2 * 2 + 1, (int64_t)kmax + 1) + 8;
  const int64_t items = (int64_t)seg::kG * seg::kMaxVirt;
  return seg::kTickBytes + sizeof(double) * static_cast<size_t>((items + seg::kG) * nv);
}
