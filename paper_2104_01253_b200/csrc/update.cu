// K2: projection updates (the reference's MvTimesMatAddMv, kernels.py:63-84).
//
// kls_dcgs2_update fuses the two MvTimesMatAddMv calls of a DCGS2 Arnoldi
// step (arnoldi.py:389-391 and :415-420; QR form ortho.py:396-398, 371-375)
// into one streaming pass over Q(:, 0:j):
//     u     = w - Q c             (delayed reorthogonalisation)
//     q_j   = u / alpha           (lagged normalisation)   -> Q(:, j)
//     w'    = aw / alpha - (Q t(0:j) + q_j t_j)            -> w (in place)
// HBM traffic 8 m (j + 4): Q once, w, aw, and the two writes.
//
// kls_mv_times_mat_add_mv is the generic Y <- scale Y + sign B S for one or
// two right-hand columns, optionally returning ||Y(:, l-1)||^2 of the result
// (fused norm for the CGS2 comparator and the DCGS2 flush).
#include "reduce.cuh"
#include "seg.cuh"
#include "tma.cuh"

#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace {

using namespace kls;

constexpr int kCols = 4;        // Q columns streamed together

// Small host coefficient vectors travel inside the launch (kernel parameter
// space, up to 32 KB on sm_70+ with CUDA >= 12.1) instead of a separate H2D
// copy: one API call per update.  __grid_constant__ lets the kernel index the
// pack in place.  NC == 0 selects the device-pointer variant.
template <int NC>
struct CoefPack {
  double v[NC > 0 ? NC : 1];
};
constexpr int kUpdRP = 2;       // row pairs per lane per chunk
constexpr int kUpdBlocksPerSm = 3;
constexpr int kUpdVirt = 148;  // virtual CTAs per segment of the fused-norm update

struct UpdParams {
  double* Q;
  int64_t ldq;
  int64_t m;
  int32_t j;
  double* w;
  const double* aw;
  const double* coef;  // c[0:j], t[0:j+1]
  double alpha;
  int32_t divide;      // aw / alpha (Arnoldi) or aw as is (QR)
  const double* alpha_dev;  // when set, alpha is read from device memory
  double* w_out;            // where w' goes (== w for the in-place update)
  int64_t m_global;         // variant choice (the same on every rank)
};

template <int RP, bool CHECK>
__device__ __forceinline__ void upd_chunk(const UpdParams& p, const double2* sct, double tj,
                                          double alpha, int64_t wbase, int lane) {
  double2 ac[RP], at[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    ac[r] = make_double2(0.0, 0.0);
    at[r] = make_double2(0.0, 0.0);
  }
  for (int k0 = 0; k0 < p.j; k0 += kCols) {
    double2 q[kCols][RP];
#pragma unroll
    for (int cc = 0; cc < kCols; ++cc) {
      if (k0 + cc < p.j) {
        const double* col = p.Q + static_cast<int64_t>(k0 + cc) * p.ldq;
#pragma unroll
        for (int r = 0; r < RP; ++r) q[cc][r] = load_pair<CHECK>(col, wbase + 64 * r + 2 * lane, p.m);
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) q[cc][r] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int cc = 0; cc < kCols; ++cc) {
      const double2 ct = sct[k0 + cc];  // zero-padded past j
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        ac[r].x = fma(q[cc][r].x, ct.x, ac[r].x);
        ac[r].y = fma(q[cc][r].y, ct.x, ac[r].y);
        at[r].x = fma(q[cc][r].x, ct.y, at[r].x);
        at[r].y = fma(q[cc][r].y, ct.y, at[r].y);
      }
    }
  }
  double* qout = p.Q + static_cast<int64_t>(p.j) * p.ldq;
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    const int64_t row = wbase + 64 * r + 2 * lane;
    const double2 w = load_pair_rw<CHECK>(p.w, row, p.m);
    const double2 a = load_pair<CHECK>(p.aw, row, p.m);
    double2 qn, wn;
    qn.x = (w.x - ac[r].x) / alpha;
    qn.y = (w.y - ac[r].y) / alpha;
    const double ax = p.divide ? a.x / alpha : a.x;
    const double ay = p.divide ? a.y / alpha : a.y;
    wn.x = ax - fma(qn.x, tj, at[r].x);
    wn.y = ay - fma(qn.y, tj, at[r].y);
    store_pair<CHECK>(qout, row, p.m, qn);
    store_pair<CHECK>(p.w_out, row, p.m, wn);
  }
}

template <int RP, int NC>
__global__ void __launch_bounds__(kThreads, kUpdBlocksPerSm)
    dcgs2_update_kernel(UpdParams p, const __grid_constant__ CoefPack<NC> pk) {
  extern __shared__ double2 sct[];  // (c_k, t_k), padded to a multiple of kCols
  pdl_wait();  // coefficients from the preceding Gram kernel
  const double* coef = NC > 0 ? pk.v : p.coef;
  const int jpad = (p.j + kCols - 1) / kCols * kCols;
  for (int k = threadIdx.x; k < jpad; k += kThreads)
    sct[k] = k < p.j ? make_double2(coef[k], coef[p.j + k]) : make_double2(0.0, 0.0);
  const double tj = coef[2 * p.j];
  const double alpha = p.alpha_dev != nullptr ? *p.alpha_dev : p.alpha;
  __syncthreads();
  constexpr int64_t WROWS = 64 * RP;
  constexpr int64_t CROWS = WROWS * kWarps;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (p.m + CROWS - 1) / CROWS;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t cbase = ch * CROWS;
    const int64_t wbase = cbase + warp * WROWS;
    if (cbase + CROWS <= p.m)
      upd_chunk<RP, false>(p, sct, tj, alpha, wbase, lane);
    else
      upd_chunk<RP, true>(p, sct, tj, alpha, wbase, lane);
  }
  pdl_trigger();
}

// Small-m K2 (global m <= kUpdSmallRows): one 64-row block per CTA, the 8
// warps splitting the basis columns (k = w, w+8, ...) so every warp has all
// its loads in flight at once; the warps' partial Q c and Q t are combined in
// fixed warp order through shared memory, then the row arithmetic of
// upd_chunk.  A 1e4-row update spreads over ~150 SMs instead of 10.
constexpr int64_t kUpdSmallRows = 1 << 16;  // scripts/small_probe.py

template <int NC>
__global__ void __launch_bounds__(kThreads) dcgs2_update_small_kernel(
    UpdParams p, const __grid_constant__ CoefPack<NC> pk) {
  extern __shared__ double2 sct[];  // (c_k, t_k), padded to a multiple of kCols
  __shared__ double2 part[kWarps][2][32];
  pdl_wait();  // coefficients from the preceding Gram kernel
  const double* coef = NC > 0 ? pk.v : p.coef;
  const int jpad = (p.j + kCols - 1) / kCols * kCols;
  for (int k = threadIdx.x; k < jpad; k += kThreads)
    sct[k] = k < p.j ? make_double2(coef[k], coef[p.j + k]) : make_double2(0.0, 0.0);
  const double tj = coef[2 * p.j];
  const double alpha = p.alpha_dev != nullptr ? *p.alpha_dev : p.alpha;
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* qout = p.Q + static_cast<int64_t>(p.j) * p.ldq;
  const int64_t nblk = (p.m + 63) / 64;
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    const int64_t row = b * 64 + 2 * lane;
    const bool full = b * 64 + 64 <= p.m;
    double2 ac = make_double2(0.0, 0.0), at = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int k = warp; k < p.j; k += kWarps) {
      const double* col = p.Q + static_cast<int64_t>(k) * p.ldq;
      const double2 q = full ? load_pair<false>(col, row, p.m) : load_pair<true>(col, row, p.m);
      const double2 ct = sct[k];
      ac.x = fma(q.x, ct.x, ac.x);
      ac.y = fma(q.y, ct.x, ac.y);
      at.x = fma(q.x, ct.y, at.x);
      at.y = fma(q.y, ct.y, at.y);
    }
    part[warp][0][lane] = ac;
    part[warp][1][lane] = at;
    __syncthreads();
    if (warp == 0) {
      double2 sc = make_double2(0.0, 0.0), stt = make_double2(0.0, 0.0);
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        sc.x += part[w][0][lane].x;
        sc.y += part[w][0][lane].y;
        stt.x += part[w][1][lane].x;
        stt.y += part[w][1][lane].y;
      }
      const double2 w = full ? load_pair_rw<false>(p.w, row, p.m) : load_pair_rw<true>(p.w, row, p.m);
      const double2 a = full ? load_pair<false>(p.aw, row, p.m) : load_pair<true>(p.aw, row, p.m);
      double2 qn, wn;
      qn.x = (w.x - sc.x) / alpha;
      qn.y = (w.y - sc.y) / alpha;
      const double ax = p.divide ? a.x / alpha : a.x;
      const double ay = p.divide ? a.y / alpha : a.y;
      wn.x = ax - fma(qn.x, tj, stt.x);
      wn.y = ay - fma(qn.y, tj, stt.y);
      if (full) {
        store_pair<false>(qout, row, p.m, qn);
        store_pair<false>(p.w_out, row, p.m, wn);
      } else {
        store_pair<true>(qout, row, p.m, qn);
        store_pair<true>(p.w_out, row, p.m, wn);
      }
    }
    __syncthreads();
  }
  pdl_trigger();
}

// TMA-staged K2: a producer warp streams 4-column x 1024-row tiles of Q and
// the chunk's w / aw rows into shared memory with cp.async.bulk (mbarrier
// completion, 4-stage ring + double-buffered vector slot); 8 consumer warps
// accumulate Q c and Q t from shared memory and write q_j and w' with
// 128-bit stores.  Same per-row arithmetic and order as the LDG kernel, so
// both variants give bitwise-identical results.
constexpr int kUR = 1024;            // rows per chunk
constexpr int kUStages = 4;
constexpr int kUThreads = (kWarps + 1) * 32;

// Optional second job of the streaming update (GMRES's per-column backward
// error, gmres.py:166-172): xout = x + Q(:, 0:q) y for an earlier column's
// least-squares y, formed from the same Q tiles (q <= j) with
// mtm_chunk's per-row operation sequence (column groups of 4, one fma per
// column, q and y read as 0 past column q within the last group), so xout
// is bit-identical to kls_mv_times_mat_add_mv(x + Q y).
constexpr int kCombMax = 64;
struct CombPack {
  const double* x;
  double* xout;
  int32_t q;
  double y[kCombMax];
};
struct CombNone {};

template <int NC, bool COMB = false>
__global__ void __launch_bounds__(kUThreads, 1)
    dcgs2_update_tma_kernel(UpdParams p, const __grid_constant__ CoefPack<NC> pk,
                            const __grid_constant__ typename std::conditional<COMB, CombPack, CombNone>::type cb) {
  using namespace kls::tma;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kUStages;
  uint64_t* xfull = empty + kUStages;
  uint64_t* xempty = xfull + 2;
  const int jpad = (p.j + kCols - 1) / kCols * kCols;
  double2* sct = reinterpret_cast<double2*>(smem + 256);
  double* qring = reinterpret_cast<double*>(sct + jpad + 1);
  double* xbuf = qring + static_cast<size_t>(kUStages) * kCols * kUR;

  const double* coef = NC > 0 ? pk.v : p.coef;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ng = (p.j + kCols - 1) / kCols;
  const int64_t m64 = p.m & ~static_cast<int64_t>(63);  // chunks: ChunkWalk (tma.cuh)
  if (threadIdx.x == 0) {
    for (int s = 0; s < kUStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(xfull + s, 1);
      mbar_init(xempty + s, kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kWarps) {
    if (lane == 0) {
      uint32_t use = 0, xuse = 0;
      int64_t row, nr;
      for (ChunkWalk<kUR> cw(m64); cw.next(row, nr); ++xuse) {
        const uint32_t bytes = static_cast<uint32_t>(nr) * sizeof(double);
        const int xs = xuse & 1;
        if (xuse >= 2) mbar_wait(xempty + xs, ((xuse >> 1) - 1) & 1);
        mbar_expect_tx(xfull + xs, 2u * bytes);
        bulk_g2s(xbuf + (static_cast<size_t>(xs) * 2) * kUR, p.w + row, bytes, xfull + xs);
        bulk_g2s(xbuf + (static_cast<size_t>(xs) * 2 + 1) * kUR, p.aw + row, bytes, xfull + xs);
        for (int g = 0; g < ng; ++g, ++use) {
          const int s = use % kUStages;
          const uint32_t round = use / kUStages;
          if (round >= 1) mbar_wait(empty + s, (round - 1) & 1);
          const int ncols = min(kCols, p.j - g * kCols);
          mbar_expect_tx(full + s, static_cast<uint32_t>(ncols) * bytes);
          for (int cc = 0; cc < ncols; ++cc)
            bulk_g2s(qring + (static_cast<size_t>(s) * kCols + cc) * kUR,
                     p.Q + static_cast<int64_t>(g * kCols + cc) * p.ldq + row, bytes, full + s);
        }
      }
    }
    return;
  }
  // consumers: the coefficients come from the preceding Gram kernel (PDL);
  // the producer above streams Q, w and aw meanwhile (none of which it writes)
  pdl_wait();
  for (int k = threadIdx.x; k < jpad; k += kWarps * 32)
    sct[k] = k < p.j ? make_double2(coef[k], coef[p.j + k]) : make_double2(0.0, 0.0);
  const double tj = coef[2 * p.j];
  const double alpha = p.alpha_dev != nullptr ? *p.alpha_dev : p.alpha;
  asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
  constexpr int RP = 2;
  const int64_t wrow = warp * (64 * RP);
  double* qout = p.Q + static_cast<int64_t>(p.j) * p.ldq;
  uint32_t use = 0, xuse = 0;
  int64_t crow, nr;  // nr: a multiple of 64; rows past it are computed but not stored
  for (ChunkWalk<kUR> cw(m64); cw.next(crow, nr); ++xuse) {
    double2 ac[RP], at[RP], xc[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      ac[r] = make_double2(0.0, 0.0);
      at[r] = make_double2(0.0, 0.0);
      xc[r] = make_double2(0.0, 0.0);
    }
    for (int g = 0; g < ng; ++g, ++use) {
      const int s = use % kUStages;
      mbar_wait(full + s, (use / kUStages) & 1);
      const double* qs = qring + static_cast<size_t>(s) * kCols * kUR;
      double2 q[kCols][RP];
#pragma unroll
      for (int cc = 0; cc < kCols; ++cc) {
        if (g * kCols + cc < p.j) {
#pragma unroll
          for (int r = 0; r < RP; ++r)
            q[cc][r] = *reinterpret_cast<const double2*>(qs + cc * kUR + wrow + 64 * r + 2 * lane);
        } else {
#pragma unroll
          for (int r = 0; r < RP; ++r) q[cc][r] = make_double2(0.0, 0.0);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);
#pragma unroll
      for (int cc = 0; cc < kCols; ++cc) {
        const double2 ct = sct[g * kCols + cc];
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          ac[r].x = fma(q[cc][r].x, ct.x, ac[r].x);
          ac[r].y = fma(q[cc][r].y, ct.x, ac[r].y);
          at[r].x = fma(q[cc][r].x, ct.y, at[r].x);
          at[r].y = fma(q[cc][r].y, ct.y, at[r].y);
        }
      }
      if constexpr (COMB) {
        if (g * kCols < cb.q) {  // mtm_chunk's groups over the first q columns
#pragma unroll
          for (int cc = 0; cc < kCols; ++cc) {
            const bool in = g * kCols + cc < cb.q;
            const double yv = in ? cb.y[g * kCols + cc] : 0.0;
#pragma unroll
            for (int r = 0; r < RP; ++r) {
              xc[r].x = fma(in ? q[cc][r].x : 0.0, yv, xc[r].x);
              xc[r].y = fma(in ? q[cc][r].y : 0.0, yv, xc[r].y);
            }
          }
        }
      }
    }
    const int xs = xuse & 1;
    mbar_wait(xfull + xs, (xuse >> 1) & 1);
    const double* xb = xbuf + static_cast<size_t>(xs) * 2 * kUR;
    double2 wv[RP], av[RP];
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      wv[r] = *reinterpret_cast<const double2*>(xb + wrow + 64 * r + 2 * lane);
      av[r] = *reinterpret_cast<const double2*>(xb + kUR + wrow + 64 * r + 2 * lane);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(xempty + xs);
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      if (wrow + 64 * r >= nr) continue;
      const int64_t row = crow + wrow + 64 * r + 2 * lane;
      double2 qn, wn;
      qn.x = (wv[r].x - ac[r].x) / alpha;
      qn.y = (wv[r].y - ac[r].y) / alpha;
      const double ax = p.divide ? av[r].x / alpha : av[r].x;
      const double ay = p.divide ? av[r].y / alpha : av[r].y;
      wn.x = ax - fma(qn.x, tj, at[r].x);
      wn.y = ay - fma(qn.y, tj, at[r].y);
      *reinterpret_cast<double2*>(qout + row) = qn;
      *reinterpret_cast<double2*>(p.w_out + row) = wn;
      if constexpr (COMB) {
        const double2 xv = ld_stream2(cb.x + row);
        *reinterpret_cast<double2*>(cb.xout + row) = make_double2(xv.x + xc[r].x, xv.y + xc[r].y);
      }
    }
  }
  if (m64 < p.m && blockIdx.x == gridDim.x - 1) {
    upd_chunk<RP, true>(p, sct, tj, alpha, m64 + wrow, lane);
    if constexpr (COMB) {  // the < 64 tail rows of xout, one per lane (warp 0)
      if (warp == 0)
        for (int64_t i = m64 + lane; i < p.m; i += 32) {
          double a = 0.0;
          for (int k0 = 0; k0 < cb.q; k0 += kCols)
#pragma unroll
            for (int cc = 0; cc < kCols; ++cc) {
              const bool in = k0 + cc < cb.q;
              a = fma(in ? __ldg(p.Q + static_cast<int64_t>(k0 + cc) * p.ldq + i) : 0.0,
                      in ? cb.y[k0 + cc] : 0.0, a);
            }
          cb.xout[i] = __ldg(cb.x + i) + a;
        }
    }
  }
  pdl_trigger();
}

// ---------------------------------------------------------------------------
// generic Y <- scale * Y + sign * B S   (l = 1 or 2 columns of Y)

struct MtmParams {
  double* Y;
  int64_t ldy;
  int64_t m;
  int32_t l;
  const double* B;
  int64_t ldb;
  int32_t k;
  const double* S;  // k x l column-major, ld = k
  double sign;
  double scale;
  double* nrm_out;  // ||Y(:, l-1)||^2 after the update, or nullptr
};

template <int L, bool CHECK>
__device__ __forceinline__ void mtm_chunk(const MtmParams& p, const double* ss, int64_t wbase,
                                          int lane, double& nrm) {
  constexpr int RP = kUpdRP;
  double2 acc[L][RP];
#pragma unroll
  for (int t = 0; t < L; ++t)
#pragma unroll
    for (int r = 0; r < RP; ++r) acc[t][r] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < p.k; k0 += kCols) {
    double2 q[kCols][RP];
#pragma unroll
    for (int cc = 0; cc < kCols; ++cc) {
      if (k0 + cc < p.k) {
        const double* col = p.B + static_cast<int64_t>(k0 + cc) * p.ldb;
#pragma unroll
        for (int r = 0; r < RP; ++r) q[cc][r] = load_pair<CHECK>(col, wbase + 64 * r + 2 * lane, p.m);
      } else {
#pragma unroll
        for (int r = 0; r < RP; ++r) q[cc][r] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int cc = 0; cc < kCols; ++cc)
#pragma unroll
      for (int t = 0; t < L; ++t) {
        const double s = ss[t * (p.k + kCols) + k0 + cc];
#pragma unroll
        for (int r = 0; r < RP; ++r) {
          acc[t][r].x = fma(q[cc][r].x, s, acc[t][r].x);
          acc[t][r].y = fma(q[cc][r].y, s, acc[t][r].y);
        }
      }
  }
#pragma unroll
  for (int t = 0; t < L; ++t) {
    double* ycol = p.Y + static_cast<int64_t>(t) * p.ldy;
#pragma unroll
    for (int r = 0; r < RP; ++r) {
      const int64_t row = wbase + 64 * r + 2 * lane;
      double2 y = load_pair_rw<CHECK>(ycol, row, p.m);
      if (p.scale != 1.0) {
        y.x *= p.scale;
        y.y *= p.scale;
      }
      if (p.k > 0) {
        y.x += p.sign * acc[t][r].x;
        y.y += p.sign * acc[t][r].y;
      }
      store_pair<CHECK>(ycol, row, p.m, y);
      if (t == L - 1) {
        nrm = fma(y.x, y.x, nrm);
        nrm = fma(y.y, y.y, nrm);
      }
    }
  }
}

template <int L, int NC>
__global__ void __launch_bounds__(kThreads, kUpdBlocksPerSm)
    mtm_kernel(MtmParams p, const __grid_constant__ CoefPack<NC> pk) {
  extern __shared__ double ss[];  // L x (k + kCols), zero-padded
  const double* S = NC > 0 ? pk.v : p.S;
  const int ldss = p.k + kCols;
  for (int i = threadIdx.x; i < L * ldss; i += kThreads) {
    const int t = i / ldss, kk = i % ldss;
    ss[i] = kk < p.k ? S[t * p.k + kk] : 0.0;
  }
  __syncthreads();
  constexpr int64_t WROWS = 64 * kUpdRP;
  constexpr int64_t CROWS = WROWS * kWarps;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double nrm = 0.0;
  const int64_t nchunks = (p.m + CROWS - 1) / CROWS;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t cbase = ch * CROWS;
    const int64_t wbase = cbase + warp * WROWS;
    if (cbase + CROWS <= p.m)
      mtm_chunk<L, false>(p, ss, wbase, lane, nrm);
    else
      mtm_chunk<L, true>(p, ss, wbase, lane, nrm);
  }
}

// The same with the fused ||Y(:, l-1)||^2, reduced over the fixed segment
// tree (seg.cuh): virtual CTA v of segment s walks the segment's chunks
// v, v + V, ...
template <int L, int NC>
__global__ void __launch_bounds__(kThreads, kUpdBlocksPerSm)
    mtm_norm_kernel(MtmParams p, const __grid_constant__ CoefPack<NC> pk,
                    const __grid_constant__ seg::SimpleArgs a) {
  extern __shared__ double ss[];  // L x (k + kCols), zero-padded
  const double* S = NC > 0 ? pk.v : p.S;
  const int ldss = p.k + kCols;
  for (int i = threadIdx.x; i < L * ldss; i += kThreads) {
    const int t = i / ldss, kk = i % ldss;
    ss[i] = kk < p.k ? S[t * p.k + kk] : 0.0;
  }
  __syncthreads();
  constexpr int64_t WROWS = 64 * kUpdRP;
  constexpr int64_t CROWS = WROWS * kWarps;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  seg::run_simple<kThreads, 1>(a, [&](int64_t r0, int64_t rows, int v, int V, double (&acc)[1]) {
    MtmParams q = p;
    q.Y = p.Y + r0;
    q.B = p.B != nullptr ? p.B + r0 : nullptr;
    q.m = rows;
    const int64_t nchunks = (rows + CROWS - 1) / CROWS;
    for (int64_t ch = v; ch < nchunks; ch += V) {
      const int64_t cbase = ch * CROWS;
      const int64_t wbase = cbase + warp * WROWS;
      if (cbase + CROWS <= rows)
        mtm_chunk<L, false>(q, ss, wbase, lane, acc[0]);
      else
        mtm_chunk<L, true>(q, ss, wbase, lane, acc[0]);
    }
  });
}

int grid_for(int64_t m, int64_t crows, int per_sm) {
  const int64_t nchunks = ceil_div(m, crows);
  int grid = static_cast<int>(std::min<int64_t>(nchunks, (int64_t)per_sm * sm_count()));
  return grid < 1 ? 1 : grid;
}

int set_smem(const void* fn, size_t smem) {
  if (smem <= 48 * 1024) return KLS_OK;
  if (smem > 227 * 1024) return fail(KLS_EINVAL, "shared memory request %zu too large", smem);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(KLS_ECUDA, "smem attribute: %s", cudaGetErrorString(e));
  return KLS_OK;
}

bool misaligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) != 0; }

// K2 variant: TMA-staged by default, KLS_UPDATE=ldg selects the LDG kernel.
bool update_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KLS_UPDATE");
    v = (e && e[0] == 'l') ? 0 : 1;
  }
  return v == 1;
}

template <int NC>
int launch_update(const UpdParams& p, const double* host_coef, cudaStream_t st) {
  static_assert(NC >= 0, "");
  CoefPack<NC> pk;
  if (NC > 0) std::memcpy(pk.v, host_coef, sizeof(double) * (2 * p.j + 1));
  // the small kernel sums a row's terms in another order than the streaming
  // kernels, so the choice follows the GLOBAL row count: every rank of a
  // sharded run (and a one-rank run) uses the same per-row arithmetic
  if (p.m_global <= kUpdSmallRows && p.j > 0 && update_tma()) {
    const size_t smem = sizeof(double2) * static_cast<size_t>((p.j + kCols - 1) / kCols * kCols + 1);
    int rc = set_smem(reinterpret_cast<const void*>(dcgs2_update_small_kernel<NC>), smem);
    if (rc) return rc;
    const int grid = grid_for(p.m, 64, 4);
    return launch_dependent(dcgs2_update_small_kernel<NC>, dim3(grid), dim3(kThreads), smem, st,
                            "dcgs2_update_small_kernel", p, pk);
  }
  const int jp = (p.j + kCols - 1) / kCols * kCols;
  const size_t tsmem = 256 + sizeof(double2) * (jp + 1) +
                       sizeof(double) * (static_cast<size_t>(kUStages) * kCols * kUR + 4 * kUR);
  if (update_tma() && p.j > 0 && p.m >= kUR && tsmem <= 227 * 1024 && !misaligned(p.Q) &&
      !misaligned(p.w) && !misaligned(p.aw) && (p.ldq % 2) == 0) {
    int rc = set_smem(reinterpret_cast<const void*>(dcgs2_update_tma_kernel<NC, false>), tsmem);
    if (rc) return rc;
    const int grid = static_cast<int>(std::min<int64_t>((p.m + kUR - 1) / kUR, sm_count()));
    return launch_dependent(dcgs2_update_tma_kernel<NC>, dim3(grid), dim3(kUThreads), tsmem, st,
                            "dcgs2_update_tma_kernel", p, pk, CombNone{});
  }
  const size_t smem = sizeof(double2) * static_cast<size_t>((p.j + kCols - 1) / kCols * kCols + 1);
  int rc = set_smem(reinterpret_cast<const void*>(dcgs2_update_kernel<kUpdRP, NC>), smem);
  if (rc) return rc;
  const int grid = grid_for(p.m, 64 * kUpdRP * kWarps, kUpdBlocksPerSm);
  return launch_dependent(dcgs2_update_kernel<kUpdRP, NC>, dim3(grid), dim3(kThreads), smem, st,
                          "dcgs2_update_kernel", p, pk);
}

int update_common(double* Q, int64_t ldq, int64_t m, int32_t j, double* w, const double* aw,
                  const double* coef, double alpha, int32_t divide, bool host,
                  const KlsSegs* segs, void* stream, const double* alpha_dev = nullptr,
                  double* w_out = nullptr) {
  if ((m > 0 && (Q == nullptr || w == nullptr || aw == nullptr)) || coef == nullptr || m < 0 ||
      j < 0 ||
      ldq < m || (ldq & 1))
    return fail(KLS_EINVAL, "dcgs2_update: bad arguments");
  if (misaligned(Q) || misaligned(w) || misaligned(aw))
    return fail(KLS_EINVAL, "dcgs2_update: operands must be 16-byte aligned");
  if (w_out != nullptr && misaligned(w_out))
    return fail(KLS_EINVAL, "dcgs2_update: w_out must be 16-byte aligned");
  seg::Layout L;
  const int rc = seg::make_layout(segs, m, L);
  if (rc) return rc;
  UpdParams p{Q, ldq, m, j, w, aw, host ? nullptr : coef, alpha, divide, alpha_dev,
              w_out != nullptr ? w_out : w, segs != nullptr ? segs->m : m};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nc = 2 * j + 1;
  if (!host) return launch_update<0>(p, nullptr, st);
  if (nc <= 32) return launch_update<32>(p, coef, st);
  if (nc <= 128) return launch_update<128>(p, coef, st);
  if (nc <= 512) return launch_update<512>(p, coef, st);
  if (nc <= 2048) return launch_update<2048>(p, coef, st);
  return fail(KLS_EINVAL, "dcgs2_update_host: 2j+1 = %d coefficients exceed the 2048 launch "
              "pack; use kls_dcgs2_update with a device array", nc);
}

template <int L, int NC>
int launch_mtm(const MtmParams& p, const double* host_s, const seg::SimpleArgs* a,
               cudaStream_t st) {
  CoefPack<NC> pk;
  if (NC > 0) std::memcpy(pk.v, host_s, sizeof(double) * p.k * L);
  const size_t smem = sizeof(double) * static_cast<size_t>(L) * (p.k + kCols);
  if (a == nullptr) {
    int rc = set_smem(reinterpret_cast<const void*>(mtm_kernel<L, NC>), smem);
    if (rc) return rc;
    const int grid = grid_for(p.m, 64 * kUpdRP * kWarps, kUpdBlocksPerSm);
    mtm_kernel<L, NC><<<grid, kThreads, smem, st>>>(p, pk);
    return check_launch("mtm_kernel");
  }
  int rc = set_smem(reinterpret_cast<const void*>(mtm_norm_kernel<L, NC>), smem);
  if (rc) return rc;
  const int grid = std::max(1, std::min(a->P.nitems, kUpdBlocksPerSm * sm_count()));
  mtm_norm_kernel<L, NC><<<grid, kThreads, smem, st>>>(p, pk, *a);
  return check_launch("mtm_norm_kernel");
}

template <int L>
int mtm_dispatch(const MtmParams& p, const double* host_s, const seg::SimpleArgs* a,
                 cudaStream_t st) {
  const int n = p.k * L;
  if (host_s == nullptr) return launch_mtm<L, 0>(p, nullptr, a, st);
  if (n <= 32) return launch_mtm<L, 32>(p, host_s, a, st);
  if (n <= 128) return launch_mtm<L, 128>(p, host_s, a, st);
  if (n <= 512) return launch_mtm<L, 512>(p, host_s, a, st);
  if (n <= 2048) return launch_mtm<L, 2048>(p, host_s, a, st);
  return fail(KLS_EINVAL, "mv_times_mat_add_mv_host: %d coefficients exceed the launch pack", n);
}

int mtm_common(double* Y, int64_t ldy, int64_t m, int32_t l, const double* B, int64_t ldb,
               int32_t k, const double* S, double sign, double scale, double* nrm_out,
               const KlsSegs* segs, void* ws, size_t ws_bytes, bool host, void* stream) {
  if ((m > 0 && Y == nullptr) || m < 0 || k < 0 || (l != 1 && l != 2) ||
      (l == 2 && (ldy < m || (ldy & 1))) ||
      (k > 0 && ((m > 0 && B == nullptr) || S == nullptr || ldb < m || (ldb & 1))))
    return fail(KLS_EINVAL, "mv_times_mat_add_mv: bad arguments (m=%lld k=%d l=%d)",
                (long long)m, k, l);
  if (misaligned(Y) || misaligned(B)) return fail(KLS_EINVAL, "mv_times_mat_add_mv: misaligned");
  MtmParams p{Y, ldy, m, l, B, ldb, k, host ? nullptr : S, sign, scale, nrm_out};
  seg::SimpleArgs a;
  const seg::SimpleArgs* ap = nullptr;
  if (nrm_out != nullptr) {
    int rc = seg::make_layout(segs, m, a.P.L);
    if (rc) return rc;
    seg::make_plan(a.P.L, 1024, kUpdVirt, a.P);
    if (ws == nullptr || seg::plan_ws_bytes(a.P, 1) > ws_bytes)
      return fail(KLS_ENOSPC, "mv_times_mat_add_mv: workspace too small for the fused norm");
    a.ws = seg::ws_of(ws, a.P.nitems, 1);
    a.d.out = nrm_out;
    a.d.xstride = 1;
    a.d.peers.world = 0;
    a.d.epoch = 0;
    a.d.err = nullptr;
    ap = &a;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const double* hs = host && k > 0 ? S : nullptr;
  if (host && k == 0) {
    static const double zero = 0.0;
    hs = &zero;
  }
  return l == 1 ? mtm_dispatch<1>(p, hs, ap, st) : mtm_dispatch<2>(p, hs, ap, st);
}

}  // namespace

// Fused DCGS2 step update (see the file header).  `coef` is a device array
// [c(0:j), t(0:j+1)] of 2j+1 doubles; column j of Q receives q_j; w is
// overwritten by the next pending vector.  divide != 0 gives the Arnoldi form
// w' = aw/alpha - ...; divide == 0 the QR form w' = a - ....
KLS_API int kls_dcgs2_update(double* Q, int64_t ldq, int64_t m, int32_t j, double* w,
                             const double* aw, const double* coef, double alpha, int32_t divide,
                             const KlsSegs* segs, void* stream) {
  return update_common(Q, ldq, m, j, w, aw, coef, alpha, divide, false, segs, stream);
}

// Same with the coefficients in HOST memory: they ride in the kernel launch
// (2j+1 <= 2048), so the step needs no separate H2D copy.
KLS_API int kls_dcgs2_update_host(double* Q, int64_t ldq, int64_t m, int32_t j, double* w,
                                  const double* aw, const double* coef_host, double alpha,
                                  int32_t divide, const KlsSegs* segs, void* stream) {
  return update_common(Q, ldq, m, j, w, aw, coef_host, alpha, divide, true, segs, stream);
}

// Same with everything on the device: coef = [c(0:j), t(0:j+1), alpha]
// (2j+2 doubles, as written by kls_dcgs2_scalars), so the update can be
// queued before the host has seen the step's scalars.  w' goes to w_out
// (w is left intact, so a speculative step can be discarded).
KLS_API int kls_dcgs2_update_dev(double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                                 double* w_out, const double* aw, const double* coef_alpha,
                                 int32_t divide, const KlsSegs* segs, void* stream) {
  if (coef_alpha == nullptr || (m > 0 && w_out == nullptr))
    return fail(KLS_EINVAL, "dcgs2_update_dev: null coefficients or output");
  return update_common(Q, ldq, m, j, const_cast<double*>(w), aw, coef_alpha, 0.0, divide, false,
                       segs, stream, coef_alpha + 2 * j + 1, w_out);
}

// Y(:, 0:l) <- scale * Y + sign * B(:, 0:k) S  with S (k x l, column-major,
// device).  When nrm_out != NULL it receives ||Y(:, l-1)||^2 of the result
// (requires ws).  Mirrors kernels.mv_times_mat_add_mv (kernels.py:63-84).
KLS_API int kls_mv_times_mat_add_mv(double* Y, int64_t ldy, int64_t m, int32_t l, const double* B,
                                    int64_t ldb, int32_t k, const double* S, double sign,
                                    double scale, double* nrm_out, const KlsSegs* segs, void* ws,
                                    size_t ws_bytes, void* stream) {
  return mtm_common(Y, ldy, m, l, B, ldb, k, S, sign, scale, nrm_out, segs, ws, ws_bytes, false,
                    stream);
}

// Same with S in HOST memory (k*l <= 2048), carried in the launch.
KLS_API int kls_mv_times_mat_add_mv_host(double* Y, int64_t ldy, int64_t m, int32_t l,
                                         const double* B, int64_t ldb, int32_t k,
                                         const double* S_host, double sign, double scale,
                                         double* nrm_out, const KlsSegs* segs, void* ws,
                                         size_t ws_bytes, void* stream) {
  return mtm_common(Y, ldy, m, l, B, ldb, k, S_host, sign, scale, nrm_out, segs, ws, ws_bytes,
                    true, stream);
}

namespace kls {

// The step update with GMRES's backward-error combination riding on it
// (plan.cu, kls_dcgs2_queue_step_be): w -> w_out and q_j as
// kls_dcgs2_update_dev, plus xout = x + Q(:, 0:q) y (y: q host doubles)
// from the same Q tiles.  Falls back to the update followed by the separate
// combination (copy + kls_mv_times_mat_add_mv_host, the same bits) where the
// streaming kernel does not apply.
int dcgs2_update_dev_comb(double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                          double* w_out, const double* aw, const double* coef_alpha,
                          const KlsSegs* segs, void* stream, const double* x, double* xout,
                          int32_t q, const double* y) {
  if (x == nullptr || xout == nullptr || y == nullptr || q < 0 || q > j)
    return fail(KLS_EINVAL, "dcgs2_update_comb: bad combination arguments");
  const int64_t m_global = segs != nullptr ? segs->m : m;
  const int jp = (j + kCols - 1) / kCols * kCols;
  const size_t tsmem = 256 + sizeof(double2) * (jp + 1) +
                       sizeof(double) * (static_cast<size_t>(kUStages) * kCols * kUR + 4 * kUR);
  const bool fused = update_tma() && j > 0 && q <= kCombMax && m >= kUR &&
                     m_global > kUpdSmallRows && tsmem <= 227 * 1024 && !misaligned(Q) &&
                     !misaligned(w) && !misaligned(aw) && !misaligned(w_out) && !misaligned(x) &&
                     !misaligned(xout) && (ldq % 2) == 0 && ldq >= m && coef_alpha != nullptr;
  if (!fused) {
    int rc = kls_dcgs2_update_dev(Q, ldq, m, j, w, w_out, aw, coef_alpha, 1, segs, stream);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (xout != x) {
      const cudaError_t e = cudaMemcpyAsync(xout, x, sizeof(double) * m, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) return fail(KLS_ECUDA, "dcgs2_update_comb: copy: %s", cudaGetErrorString(e));
    }
    if (q == 0) return KLS_OK;
    return kls_mv_times_mat_add_mv_host(xout, ldq, m, 1, Q, ldq, q, y, 1.0, 1.0, nullptr, segs,
                                        nullptr, 0, stream);
  }
  seg::Layout L;
  int rc = seg::make_layout(segs, m, L);
  if (rc) return rc;
  UpdParams p{Q, ldq, m, j, const_cast<double*>(w), aw, coef_alpha, 0.0, 1, coef_alpha + 2 * j + 1,
              w_out, m_global};
  CoefPack<0> pk;
  CombPack cb;
  cb.x = x;
  cb.xout = xout;
  cb.q = q;
  for (int i = 0; i < kCombMax; ++i) cb.y[i] = i < q ? y[i] : 0.0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rc = set_smem(reinterpret_cast<const void*>(dcgs2_update_tma_kernel<0, true>), tsmem);
  if (rc) return rc;
  const int grid = static_cast<int>(std::min<int64_t>((m + kUR - 1) / kUR, sm_count()));
  return launch_dependent(dcgs2_update_tma_kernel<0, true>, dim3(grid), dim3(kUThreads), tsmem, st,
                          "dcgs2_update_tma_kernel", p, pk, cb);
}

}  // namespace kls
