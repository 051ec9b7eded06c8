// One DCGS2 Arnoldi step in ONE persistent launch for banded ELL operators:
//
//     K2(j)    q_j = (w - Q c)/alpha -> Q(:, j),  w' = aw/alpha - (Q t + q_j t_j)
//     K3       Aw' = A w'                        (ELL, half bandwidth h rows)
//     K1(j+1)  g = [Q(:, 0:j+1), w']^T [w', Aw'],  ||Aw'||^2,
//              fixed-tree reduction and the device scalar step of step j+1
//
// (arnoldi.py:389-391, 415-420, problems.py:127-136, arnoldi.py:362-370, 414).
//
// Why: the unfused step streams Q(:, 0:j) from HBM twice (K2, then K1 of the
// next step) with two launch boundaries and a full operator pass between
// them.  Here a CTA takes one row chunk (an item of the Gram plan: 1024 rows)
// through all three stages back to back: the K1 pass re-reads the chunk's Q
// tiles microseconds after the K2 pass streamed them, so they come from L2
// (the K2 copies carry an L2 evict_last hint, the K1 copies evict_first), w'
// and Aw' of the chunk never leave shared memory for the Gram pass, and the
// only cross-CTA dependency -- the operator's halo of h rows -- is a per-
// chunk release/acquire flag.  HBM traffic per step drops from
// ~8m(2j + 8) + ELL to ~8m(j + 5) + ELL.
//
// Chunks are dealt round-robin (item it -> CTA it % grid), so the halo of a
// chunk lies in chunks other CTAs process in the same round: the waits are
// short, and with at most `grid - 1` chunks of halo on each side a chain of
// waits always ends (every wait is on an item of lower round or of the same
// round on a CTA that does not wait back) -- the launch needs all its CTAs
// co-resident, which one CTA per SM and grid <= SM count guarantee.
//
// Arithmetic: K2's per-row expressions are those of dcgs2_update_tma_kernel,
// the ELL row sums those of kls_ell_spmv, and the Gram pass accumulates a
// chunk exactly as gram_tma_kernel does for a one-chunk item (same warp /
// row mapping, column groups, butterfly, warp-order item sum), and the plan
// is the one launch_gram uses at this size (seg::make_plan with 1024-row
// items).  So the fused step is bitwise identical to the three unfused
// launches, on one rank and -- through the segment tree -- on any number.
#include "gram.cuh"
#include "tma.cuh"

#include <cstdlib>
#include <mutex>
#include <map>

namespace kls {
namespace fused {
namespace {

using namespace kls::tma;
using gram::kG;  // 4 Q columns per stage

constexpr int kR = 1024;  // rows per chunk (= Gram item)
constexpr int kRP = 2;    // row pairs per lane: 8 warps x 64 x 2 = 1024
constexpr int kNX = 2;           // Gram right-hand vectors: w', Aw'
constexpr int kV = kG * kNX;     // outputs per column group
constexpr int kMaxCols = 256;    // Gram columns (j + 1) per launch
constexpr uint64_t kTimeoutNs = 4ull * 1000 * 1000 * 1000;

struct Params {
  double* Q;
  int64_t ldq;
  int64_t m;  // rows (one rank)
  int32_t j;  // K2 writes Q(:, j); the Gram pass covers j + 1 columns
  const double* coef;  // [c(0:j), t(0:j+1), alpha] of step j (read at launch start)
  const double* w;
  const double* aw;
  double* w_out;
  double* aw_out;
  const int32_t* ecol;
  const double* eval;
  const uint8_t* elen;
  int32_t width;
  int64_t eld;
  int64_t reach;  // max |col - row| + 1
  unsigned* flags;  // per item: epoch once its w' rows are stored
  unsigned epoch;
  int* err;
  seg::Plan P;
  seg::Ws ws;
  seg::Dest d;
  double* coef_out;  // the next step's coefficients (may alias coef)
  double* gout;
  int32_t nv;
  int32_t hints;  // L2 cache hints on the two Q passes (KLS_FUSED_HINT=0: none)
  int32_t dbg;  // experiments (KLS_FUSED_DBG bits): 1 no halo wait, 2 no publish fence
  int64_t* trace;  // experiments: per item [start, K2 done, halo ready, K3 done, K1 done] (ns)
};

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Rows of item `it`: [row, row + nr) with nr a multiple of 64 (segment-
// relative, ChunkWalk's schedule for a one-chunk item), plus the segment's
// < 64 tail rows [tail0, tail1) when the item is the segment's last.
struct Chunk {
  int64_t base, row, nr, tail0, tail1;
};
__device__ __forceinline__ Chunk chunk_of(const seg::Plan& P, int it) {
  int s, v, Vn;
  seg::item_of(P, it, s, v, Vn);
  Chunk c;
  c.base = P.L.off[s];
  const int64_t rows = P.L.off[s + 1] - c.base;
  const int64_t m64 = rows & ~static_cast<int64_t>(63);
  ChunkWalk<kR> cw(m64, Vn, v, int64_t(1) << 40);
  int64_t r = 0, nr = 0;
  if (!cw.next(r, nr)) {
    r = m64;
    nr = 0;
  }
  c.row = c.base + r;
  c.nr = nr;
  c.tail0 = c.tail1 = c.base + rows;
  if (v == Vn - 1 && m64 < rows) c.tail0 = c.base + m64;
  return c;
}

// The item holding local row x (0 <= x < m).
__device__ __forceinline__ int item_of_row(const seg::Plan& P, int64_t x) {
  int s = 0;
  while (s + 1 < P.L.nseg && P.L.off[s + 1] <= x) ++s;
  const int Vn = P.ibase[s + 1] - P.ibase[s];
  const int64_t rows = P.L.off[s + 1] - P.L.off[s];
  const int64_t m64 = rows & ~static_cast<int64_t>(63);
  const int64_t q = m64 / kR / Vn;
  const int64_t per = q >= 1 ? kR : ((m64 / 64 + Vn - 1) / Vn) * 64;
  int64_t v = per > 0 ? (x - P.L.off[s]) / per : 0;
  if (v > Vn - 1) v = Vn - 1;
  return P.ibase[s] + static_cast<int>(v);
}

__device__ __forceinline__ int ld_na_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<int>(v);
}
__device__ __forceinline__ int32_t ld_na_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_na_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// ELL rows of one thread in the K3 stage: the entries of all its rows are
// fetched up front (before the halo wait -- the operator's arrays are never
// written), then every gather is in flight at once.  Row sums in
// kls_ell_spmv's order (products k < n, reduceat pairing).
template <int W, int NR>
struct EllRows {
  int n[NR];
  int32_t c[NR][W];
  double v[NR][W];

  __device__ __forceinline__ void fetch(const Params& p, const int64_t (&row)[NR],
                                        const bool (&on)[NR]) {
#pragma unroll
    for (int i = 0; i < NR; ++i) n[i] = on[i] ? ld_na_u8(p.elen + row[i]) : 0;
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const bool e = on[i] && k < p.width;
        c[i][k] = e ? ld_na_s32(p.ecol + k * p.eld + row[i]) : 0;
        v[i][k] = e ? ld_na_f64(p.eval + k * p.eld + row[i]) : 0.0;
      }
  }

  __device__ __forceinline__ void apply(const double* x, double (&y)[NR]) const {
    double pr[NR][W];
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
      for (int k = 0; k < W; ++k) pr[i][k] = k < n[i] ? __dmul_rn(v[i][k], __ldcg(x + c[i][k])) : 0.0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      double acc = 0.0;
      if (n[i] > 0) {
        double r = -0.0;
#pragma unroll
        for (int k = 1; k < W; ++k)
          if (k < n[i]) r = __dadd_rn(r, pr[i][k]);
        acc = __dadd_rn(pr[i][0], r);
      }
      y[i] = acc;
    }
  }
};

// Warp roles (one CTA per SM).  A chunk's update streams Q from HBM; its
// operator product is a chain of dependent gathers (entries, then w' rows)
// that under a saturated memory system costs microseconds of latency; its
// Gram pass re-reads Q from L2.  Run back to back in one group of warps the
// three leave HBM idle most of the time, so they run concurrently on
// consecutive chunks of the CTA's list:
//   warps 0-7   (G) operator product + Gram pass of chunk k-1 -- the Gram
//               pass with gram_tma_kernel's 8-warp row mapping (bitwise);
//   warps 8-11  (U) update of chunk k (4 warps x 2 halves of 512 rows), at
//               most one chunk ahead of G so G's Q tiles are still in L2;
//   warp 12     TMA producer of U's ring (Q tiles from HBM, evict_last);
//   warp 13     TMA producer of G's ring (the same tiles from L2, evict_first).
constexpr int kGW = 8;                 // product + Gram warps
constexpr int kUW = 4;                 // update warps
constexpr int kGT = kGW * 32;
constexpr int kUT = kUW * 32;
constexpr int kPA = kGW + kUW;         // producer warp of ring A
constexpr int kPC = kPA + 1;           // producer warp of ring C
constexpr int kThreadsWS = (kPC + 1) * 32;
constexpr int kSA = 3, kSC = 2;        // ring stages (4 columns x 1024 rows each)

__device__ __forceinline__ void ubar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kUT) : "memory");
}

template <int W>
__global__ void __launch_bounds__(kThreadsWS, 1) dcgs2_fused_kernel(Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double sx[kGW][kNX + 1];
  __shared__ double s_red[kThreadsWS];
  __shared__ int s_flag, s_ok, s_fin;
  __shared__ volatile int s_gdone;  // chunks G has finished
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem);
  uint64_t* emptyA = fullA + kSA;
  uint64_t* fullC = emptyA + kSA;
  uint64_t* emptyC = fullC + kSC;
  const int j = p.j;
  const int k1 = j + 1;                       // Gram columns
  const int ngA = (j + kG - 1) / kG;          // ring groups per pass (columns < j)
  const int ngC = (k1 + kG - 1) / kG;         // Gram column groups
  const int jpad = ngA * kG;
  const int stride = ngC * kV;                // per-warp accumulators
  double2* sct = reinterpret_cast<double2*>(smem + 256);
  double* ringA = reinterpret_cast<double*>(sct + jpad + 1);
  double* ringC = ringA + static_cast<size_t>(kSA) * kG * kR;
  double* abuf = ringC + static_cast<size_t>(kSC) * kG * kR;  // Aw' of G's chunk
  double* sacc = abuf + kR;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const int nq = k1 * kNX;

  if (tid == 0) {
    for (int s = 0; s < kSA; ++s) {
      mbar_init(fullA + s, 1);
      mbar_init(emptyA + s, kUW);
    }
    for (int s = 0; s < kSC; ++s) {
      mbar_init(fullC + s, 1);
      mbar_init(emptyC + s, kGW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_fin = 0;
    s_gdone = 0;
  }
  for (int i = tid; i < (kSA + kSC) * kG * kR / 2; i += blockDim.x)
    reinterpret_cast<double2*>(ringA)[i] = make_double2(0.0, 0.0);
  for (int i = tid; i < kR / 2; i += blockDim.x)
    reinterpret_cast<double2*>(abuf)[i] = make_double2(0.0, 0.0);
  for (int i = tid; i < kGW * stride; i += blockDim.x) sacc[i] = 0.0;
  for (int k = tid; k < jpad; k += blockDim.x)
    sct[k] = k < j ? make_double2(0.0, 0.0) : make_double2(0.0, 0.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  // everything below reads what the preceding step wrote (w, aw, Q(:, j-1),
  // coef): the whole CTA waits for it
  pdl_wait();

  if (warp == kPA || warp == kPC) {
    // ---- producers ----------------------------------------------------------
    if (lane == 0) {
      const bool A = warp == kPA;
      const uint64_t pol = A ? policy_evict_last() : policy_evict_first();
      const int S = A ? kSA : kSC;
      double* ring = A ? ringA : ringC;
      uint64_t* full = A ? fullA : fullC;
      uint64_t* empty = A ? emptyA : emptyC;
      uint32_t use = 0;
      for (int it = blockIdx.x; it < p.P.nitems; it += gridDim.x) {
        const Chunk c = chunk_of(p.P, it);
        const uint32_t bytes = static_cast<uint32_t>(c.nr) * sizeof(double);
        for (int g = 0; g < ngA; ++g, ++use) {
          const int st = use % S;
          const uint32_t round = use / S;
          if (round >= 1) mbar_wait(empty + st, (round - 1) & 1);
          const int ncols = min(kG, j - g * kG);
          mbar_expect_tx(full + st, static_cast<uint32_t>(ncols) * bytes);
          if (bytes)
            for (int cc = 0; cc < ncols; ++cc) {
              double* dst = ring + (static_cast<size_t>(st) * kG + cc) * kR;
              const double* src = p.Q + static_cast<int64_t>(g * kG + cc) * p.ldq + c.row;
              if (p.hints)
                bulk_g2s_hint(dst, src, bytes, full + st, pol);
              else
                bulk_g2s(dst, src, bytes, full + st);
            }
        }
      }
    }
  } else if (warp >= kGW) {
    // ---- U: the update, one chunk ahead of G ----------------------------------
    const int ut = tid - kGT;  // 0..127
    const int uw = warp - kGW;
    for (int k = ut; k < jpad; k += kUT)
      sct[k] = k < j ? make_double2(p.coef[k], p.coef[j + k]) : make_double2(0.0, 0.0);
    const double tj = p.coef[2 * j];
    const double alpha = p.coef[2 * j + 1];
    ubar();
    double* qout = p.Q + static_cast<int64_t>(j) * p.ldq;
    uint32_t use = 0;
    int k = 0;
    for (int it = blockIdx.x; it < p.P.nitems; it += gridDim.x, ++k) {
      const Chunk c = chunk_of(p.P, it);
      if (p.trace != nullptr && ut == 0) p.trace[8 * it] = peer::now_ns();
      if (ut == 0)  // G has finished chunk k - 2 (so G's tiles of k - 1 stay in L2)
        while (s_gdone < k - 1) __nanosleep(64);
      ubar();
      if (p.trace != nullptr && ut == 0) p.trace[8 * it + 1] = peer::now_ns();
      // rows h * 512 + uw * 128 + 64 r + 2 lane: per-row arithmetic of K2
      double2 ac[2][kRP], at[2][kRP];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int r = 0; r < kRP; ++r) {
          ac[h][r] = make_double2(0.0, 0.0);
          at[h][r] = make_double2(0.0, 0.0);
        }
      for (int g = 0; g < ngA; ++g, ++use) {
        const int st = use % kSA;
        mbar_wait(fullA + st, (use / kSA) & 1);
        const double* qs = ringA + static_cast<size_t>(st) * kG * kR;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2 q[kG][kRP];
#pragma unroll
          for (int cc = 0; cc < kG; ++cc)
#pragma unroll
            for (int r = 0; r < kRP; ++r)
              q[cc][r] = g * kG + cc < j ? *reinterpret_cast<const double2*>(
                                               qs + cc * kR + h * 512 + uw * 128 + 64 * r + 2 * lane)
                                         : make_double2(0.0, 0.0);
#pragma unroll
          for (int cc = 0; cc < kG; ++cc) {
            const double2 ct = sct[g * kG + cc];
#pragma unroll
            for (int r = 0; r < kRP; ++r) {
              ac[h][r].x = fma(q[cc][r].x, ct.x, ac[h][r].x);
              ac[h][r].y = fma(q[cc][r].y, ct.x, ac[h][r].y);
              at[h][r].x = fma(q[cc][r].x, ct.y, at[h][r].x);
              at[h][r].y = fma(q[cc][r].y, ct.y, at[h][r].y);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(emptyA + st);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int r = 0; r < kRP; ++r) {
          const int64_t lr = h * 512 + uw * 128 + 64 * r + 2 * lane;
          if (lr >= c.nr) continue;
          const double2 wv = ld_stream2(p.w + c.row + lr);   // inputs: never
          const double2 av = ld_stream2(p.aw + c.row + lr);  // written here
          double2 qn, wn;
          qn.x = (wv.x - ac[h][r].x) / alpha;
          qn.y = (wv.y - ac[h][r].y) / alpha;
          const double ax = av.x / alpha;
          const double ay = av.y / alpha;
          wn.x = ax - fma(qn.x, tj, at[h][r].x);
          wn.y = ay - fma(qn.y, tj, at[h][r].y);
          *reinterpret_cast<double2*>(qout + c.row + lr) = qn;
          *reinterpret_cast<double2*>(p.w_out + c.row + lr) = wn;
        }
      // the segment's < 64 tail rows (the LDG update of upd_chunk)
      if (c.tail0 < c.tail1 && uw == 0) {
        for (int64_t i = c.tail0 + lane; i < c.tail1; i += 32) {
          double a1 = 0.0, a2 = 0.0;
          for (int k0 = 0; k0 < j; k0 += kG) {  // upd_chunk's order
#pragma unroll
            for (int cc = 0; cc < kG; ++cc) {
              const double qv = k0 + cc < j ? __ldg(p.Q + static_cast<int64_t>(k0 + cc) * p.ldq + i) : 0.0;
              const double2 ct = sct[k0 + cc];
              a1 = fma(qv, ct.x, a1);
              a2 = fma(qv, ct.y, a2);
            }
          }
          const double qn = (__ldg(p.w + i) - a1) / alpha;
          const double wn = __ldg(p.aw + i) / alpha - fma(qn, tj, a2);
          qout[i] = qn;
          p.w_out[i] = wn;
        }
      }
      ubar();
      if (ut == 0) {
        if (!(p.dbg & 2)) __threadfence();
        st_release_gpu(p.flags + it, p.epoch);
        if (p.trace != nullptr) p.trace[8 * it + 2] = peer::now_ns();
      }
    }
  } else {
    // ---- G: operator product + Gram pass --------------------------------------
    double* wacc = sacc + warp * stride;
    const int64_t wrow = warp * (64 * kRP);
    const double* qcol = p.Q + static_cast<int64_t>(j) * p.ldq;
    constexpr int NB = kR / kGT;  // product rows per thread
    uint32_t use = 0;
    int k = 0;
    for (int it = blockIdx.x; it < p.P.nitems; it += gridDim.x, ++k) {
      const Chunk c = chunk_of(p.P, it);
      if (p.trace != nullptr && tid == 0) p.trace[8 * it + 3] = peer::now_ns();
      // the product's entries (the operator's own arrays) while the halo lands
      EllRows<W, NB> er;
      int64_t rr[NB];
      bool on[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        rr[i] = c.row + tid + i * kGT;
        on[i] = tid + i * kGT < c.nr;
      }
      er.fetch(p, rr, on);
      {
        const int64_t r_end = c.tail1 > c.tail0 ? c.tail1 : c.row + c.nr;
        const int64_t lo = c.row - p.reach + 1 > 0 ? c.row - p.reach + 1 : 0;
        const int64_t hi = r_end + p.reach - 1 < p.m ? r_end + p.reach - 1 : p.m;
        const int ilo = item_of_row(p.P, lo), ihi = item_of_row(p.P, hi - 1);
        for (int q = ilo + tid; q <= ihi; q += kGT) {  // includes this chunk (U)
          const unsigned* f = p.flags + q;
          if (static_cast<int>(ld_acquire_gpu(f) - p.epoch) < 0) {
            const uint64_t t0 = peer::now_ns();
            while (static_cast<int>(ld_acquire_gpu(f) - p.epoch) < 0) {
              if (peer::now_ns() - t0 > kTimeoutNs) {
                atomicExch(p.err, 1);
                break;
              }
              __nanosleep(32);
            }
          }
        }
      }
      seg::gsync<kGT, 2>();
      if (p.trace != nullptr && tid == 0) p.trace[8 * it + 4] = peer::now_ns();
      {
        double y[NB];
        er.apply(p.w_out, y);
#pragma unroll
        for (int i = 0; i < NB; ++i)
          if (on[i]) {
            p.aw_out[rr[i]] = y[i];
            abuf[tid + i * kGT] = y[i];
          }
      }
      if (c.tail0 < c.tail1 && tid < 64) {  // < 64 tail rows: one per thread
        EllRows<W, 1> et;
        const int64_t r1[1] = {c.tail0 + tid};
        const bool o1[1] = {c.tail0 + tid < c.tail1};
        et.fetch(p, r1, o1);
        double y[1];
        et.apply(p.w_out, y);
        if (o1[0]) p.aw_out[r1[0]] = y[0];
      }
      seg::gsync<kGT, 2>();
      if (p.trace != nullptr && tid == 0) p.trace[8 * it + 5] = peer::now_ns();

      // K1 of step j+1 over the chunk (gram_tma_kernel's arithmetic)
      bool live[kRP];
#pragma unroll
      for (int r = 0; r < kRP; ++r) live[r] = wrow + 64 * r < c.nr;
      double ex[kNX] = {0.0, 0.0};
      double xn = 0.0;
      double2 xv[kNX][kRP];
#pragma unroll
      for (int r = 0; r < kRP; ++r) {
        const int64_t lr = wrow + 64 * r + 2 * lane;
        // w' rows: stored by U before it released this chunk's flag
        xv[0][r] = live[r] ? __ldcg(reinterpret_cast<const double2*>(p.w_out + c.row + lr))
                           : make_double2(0.0, 0.0);
        xv[1][r] = live[r] ? *reinterpret_cast<const double2*>(abuf + lr) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int r = 0; r < kRP; ++r) {
        const double2 b = xv[0][r];  // bext == x0 (w')
#pragma unroll
        for (int t = 0; t < kNX; ++t) {
          ex[t] = fma(b.x, xv[t][r].x, ex[t]);
          ex[t] = fma(b.y, xv[t][r].y, ex[t]);
        }
      }
#pragma unroll
      for (int r = 0; r < kRP; ++r) {
        xn = fma(xv[kNX - 1][r].x, xv[kNX - 1][r].x, xn);
        xn = fma(xv[kNX - 1][r].y, xv[kNX - 1][r].y, xn);
      }
      for (int g = 0; g < ngC; ++g) {
        const bool ring = g < ngA;
        int st = 0;
        const double* qs = nullptr;
        if (ring) {
          st = use % kSC;
          mbar_wait(fullC + st, (use / kSC) & 1);
          qs = ringC + static_cast<size_t>(st) * kG * kR;
        }
        double2 q[kG][kRP];
#pragma unroll
        for (int cc = 0; cc < kG; ++cc) {
          const int col = g * kG + cc;
#pragma unroll
          for (int r = 0; r < kRP; ++r) {
            const int64_t lr = wrow + 64 * r + 2 * lane;
            q[cc][r] = col < j ? *reinterpret_cast<const double2*>(qs + cc * kR + lr)
                       : col == j && live[r]
                           ? __ldcg(reinterpret_cast<const double2*>(qcol + c.row + lr))
                           : make_double2(0.0, 0.0);
          }
        }
        if (ring) {
          __syncwarp();
          if (lane == 0) mbar_arrive(emptyC + st);
          ++use;
        }
        double acc[kV];
#pragma unroll
        for (int vv = 0; vv < kV; ++vv) acc[vv] = 0.0;
#pragma unroll
        for (int cc = 0; cc < kG; ++cc)
#pragma unroll
          for (int r = 0; r < kRP; ++r)
#pragma unroll
            for (int t = 0; t < kNX; ++t) {
              acc[cc * kNX + t] = fma(q[cc][r].x, xv[t][r].x, acc[cc * kNX + t]);
              acc[cc * kNX + t] = fma(q[cc][r].y, xv[t][r].y, acc[cc * kNX + t]);
            }
        const double sred = warp_transpose_reduce<kV>(acc, lane);
        if ((lane & (32 / kV - 1)) == 0) wacc[g * kV + warp_slot<kV>(lane)] += sred;
      }
      if (c.tail0 < c.tail1) {
        // the segment's tail rows through the coherent path (written above)
        const int64_t rows = c.tail1 - c.base;
        const int64_t m64 = c.tail0 - c.base;
        const gram::GramRows gr{p.Q + c.base, p.ldq, k1, p.w_out + c.base, p.w_out + c.base,
                                p.aw_out + c.base, rows, 1};
        gram::gram_chunk<kNX, kRP, true, true>(gr, m64 + wrow, lane, wacc, ex, xn);
      }
#pragma unroll
      for (int t = 0; t < kNX; ++t) {
        const double sv = warp_sum(ex[t]);
        if (lane == 0) sx[warp][t] = sv;
      }
      {
        const double sv = warp_sum(xn);
        if (lane == 0) sx[warp][kNX] = sv;
      }
      seg::gsync<kGT, 2>();
      seg::item_store<kGT>(p.ws, it, p.nv, tid, [&](int i) {
        double t = 0.0;
        if (i < nq) {
#pragma unroll
          for (int w = 0; w < kGW; ++w) t += sacc[w * stride + i];
        } else if (i < nq + kNX) {
#pragma unroll
          for (int w = 0; w < kGW; ++w) t += sx[w][i - nq];
        } else {
#pragma unroll
          for (int w = 0; w < kGW; ++w) t += sx[w][kNX];
        }
        return t;
      });
      seg::gsync<kGT, 2>();
      for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
      __syncwarp();
      if (tid == 0) {
        s_gdone = k + 1;
        if (p.trace != nullptr) p.trace[8 * it + 6] = peer::now_ns();
      }
    }
    if (seg::finish_items<kGT, 2>(p.P, p.ws, p.nv, tid, s_red, &s_flag) && tid == 0) s_fin = 1;
  }
  pdl_trigger();
  __syncthreads();
  if (!s_fin) return;
  // gram_dst's output mapping for [Q(:, 0:k1), w']^T [w', Aw'] (+ Aw'.Aw')
  const int64_t ld = k1 + 1;
  const bool ok = seg::seg_final<kThreadsWS, 0>(p.P.L, p.ws, p.nv, p.d, tid, &s_ok, [&](int i) {
    return i < nq ? (i % kNX) * ld + i / kNX : i < nq + kNX ? (i - nq) * ld + k1 : kNX * ld;
  });
  if (ok) {
    __syncthreads();
    dcgs2_scalars_block(p.d.out, k1, 0, p.coef_out, p.gout);
  }
}

// Per (device, stream): the chunk flags (zeroed once; an epoch per launch,
// so they never need resetting) and a device error word.
struct FlagBuf {
  unsigned* flags = nullptr;
  size_t n = 0;
  unsigned epoch = 0;
  int* err = nullptr;
};
std::mutex g_mu;
std::map<std::pair<int, void*>, FlagBuf> g_flags;

int flags_for(void* stream, int nitems, FlagBuf*& out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  FlagBuf& b = g_flags[{dev, stream}];
  if (b.n < static_cast<size_t>(nitems)) {
    // a replaced buffer may still be read by queued work: keep it (leak)
    size_t n = std::max<size_t>(nitems, 4096);
    unsigned* f = nullptr;
    cudaError_t e = cudaMalloc(&f, n * sizeof(unsigned));
    if (e != cudaSuccess) return fail(KLS_ECUDA, "fused step: flag buffer: %s", cudaGetErrorString(e));
    e = cudaMemsetAsync(f, 0, n * sizeof(unsigned), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(KLS_ECUDA, "fused step: flag memset: %s", cudaGetErrorString(e));
    b.flags = f;
    b.n = n;
    b.epoch = 0;
    if (b.err == nullptr) {
      e = cudaMalloc(&b.err, sizeof(int));
      if (e == cudaSuccess) e = cudaMemsetAsync(b.err, 0, sizeof(int), static_cast<cudaStream_t>(stream));
      if (e != cudaSuccess) return fail(KLS_ECUDA, "fused step: error word: %s", cudaGetErrorString(e));
    }
  }
  ++b.epoch;
  if (b.epoch == 0x7fffffffu) {  // keep (int)(flag - epoch) comparisons exact: restart
    cudaMemsetAsync(b.flags, 0, b.n * sizeof(unsigned), static_cast<cudaStream_t>(stream));
    b.epoch = 1;
  }
  out = &b;
  return KLS_OK;
}

size_t smem_bytes(int j) {
  const int ngA = (j + kG - 1) / kG;
  const int ngC = (j + 1 + kG - 1) / kG;
  return 256 + sizeof(double2) * (ngA * kG + 1) +
         sizeof(double) * (static_cast<size_t>(kSA + kSC) * kG * kR + kR +
                           static_cast<size_t>(kGW) * ngC * kV);
}

bool fused_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KLS_FUSED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int W>
int launch_w(const Params& p, int grid, size_t smem, cudaStream_t st) {
  static size_t attr = 0;  // the largest dynamic size set so far
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(dcgs2_fused_kernel<W>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "fused step: smem attr: %s", cudaGetErrorString(e));
    attr = smem;
  }
  return launch_dependent(dcgs2_fused_kernel<W>, dim3(grid), dim3(kThreadsWS), smem, st,
                          "dcgs2_fused_kernel", p);
}

}  // namespace
}  // namespace fused

// Whether kls_dcgs2_fused_step applies to step j of this plan (one rank, a
// banded ELL operator, the chunk-item Gram tree, the basis panel and the
// shared memory within bounds).
bool dcgs2_fused_ok(const KlsStepPlan* p, int32_t j) {
  using namespace fused;
  if (!fused_enabled() || p == nullptr || p->op.kind != KLS_OP_ELL || p->op.reach < 1 ||
      p->op.width < 1 || p->op.width > 8 || p->qr || !p->divide || p->segs.world != 1 ||
      p->m != p->segs.m || p->op.m != p->m)
    return false;
  // dynamic shared memory within the 227 KB opt-in, next to ~4 KB static
  if (!gram::chunk_tree(p->segs.m) || j + 1 > kMaxCols || smem_bytes(j) > 222 * 1024) return false;
  // halo within grid - 1 chunks on each side (the wait chains end), with margin
  if (p->op.reach > static_cast<int64_t>(kR) * 32) return false;
  if ((reinterpret_cast<uintptr_t>(p->Q) & 15) || (p->ldq & 1)) return false;
  return true;
}

}  // namespace kls

using namespace kls;

// One fused DCGS2 step (file header): update of step j (w -> w_out, q_j ->
// Q(:, j)), A w_out -> aw_out, the Gram pass of step j + 1 with its reduction
// and device scalar step (-> plan->gdev, plan->cdev, plan->gout[slot]).
// Results are bitwise those of kls_dcgs2_queue_step's three launches.
static int fused_step(const KlsStepPlan* plan, int32_t j, const double* w, double* w_out,
                      const double* aw, double* aw_out, int32_t slot, int64_t* trace) {
  using namespace kls::fused;
  if (plan == nullptr || slot < 0 || slot > 1 || j < 0)
    return fail(KLS_EINVAL, "fused step: bad arguments");
  if (!dcgs2_fused_ok(plan, j)) return fail(KLS_EINVAL, "fused step: not eligible (j = %d)", j);
  if (((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(w_out) |
        reinterpret_cast<uintptr_t>(aw) | reinterpret_cast<uintptr_t>(aw_out)) & 15))
    return fail(KLS_EINVAL, "fused step: vectors must be 16-byte aligned");
  Params p;
  int rc = seg::make_layout(&plan->segs, plan->m, p.P.L);
  if (rc) return rc;
  gram::chunk_plan(p.P.L, p.P);
  p.nv = 2 * (j + 1) + 3;
  if (seg::plan_ws_bytes(p.P, p.nv) > plan->ws_bytes)
    return fail(KLS_ENOSPC, "fused step: workspace %zu bytes < %zu needed", plan->ws_bytes,
                seg::plan_ws_bytes(p.P, p.nv));
  p.ws = seg::ws_of(plan->ws, p.P.nitems, p.nv);
  FlagBuf* fb = nullptr;
  rc = flags_for(plan->stream, p.P.nitems, fb);
  if (rc) return rc;
  p.Q = plan->Q;
  p.ldq = plan->ldq;
  p.m = plan->m;
  p.j = j;
  p.coef = plan->cdev;
  p.w = w;
  p.aw = aw;
  p.w_out = w_out;
  p.aw_out = aw_out;
  p.ecol = static_cast<const int32_t*>(plan->op.p0);
  p.eval = static_cast<const double*>(plan->op.p1);
  p.elen = static_cast<const uint8_t*>(plan->op.p2);
  p.width = plan->op.width;
  p.eld = plan->op.n0;
  p.reach = plan->op.reach;
  p.flags = fb->flags;
  p.epoch = fb->epoch;
  p.err = fb->err;
  p.d.out = plan->gdev;
  p.d.xstride = 0;
  p.d.peers.world = 0;
  p.d.epoch = 0;
  p.d.err = nullptr;
  p.coef_out = plan->cdev;
  p.gout = plan->gout[slot];
  static const int hints = [] {
    const char* e = getenv("KLS_FUSED_HINT");
    return e != nullptr && e[0] == '0' ? 0 : 1;
  }();
  p.hints = hints;
  p.trace = trace;
  static const int dbg = [] {
    const char* e = getenv("KLS_FUSED_DBG");
    return e != nullptr ? atoi(e) : 0;
  }();
  p.dbg = dbg;
  const int grid = std::max(1, std::min(p.P.nitems, sm_count()));
  const size_t smem = smem_bytes(j);
  cudaStream_t st = static_cast<cudaStream_t>(plan->stream);
  switch (p.width <= 4 ? 4 : p.width) {
    case 5: return launch_w<5>(p, grid, smem, st);
    case 6: return launch_w<6>(p, grid, smem, st);
    case 7: return launch_w<7>(p, grid, smem, st);
    case 8: return launch_w<8>(p, grid, smem, st);
    default: return launch_w<4>(p, grid, smem, st);
  }
}

KLS_API int kls_dcgs2_fused_step(const KlsStepPlan* plan, int32_t j, const double* w,
                                 double* w_out, const double* aw, double* aw_out, int32_t slot) {
  return fused_step(plan, j, w, w_out, aw, aw_out, slot, nullptr);
}

// Experiments (scripts/exp/fused_probe.py): the same step recording, per
// item, %globaltimer at its start and after its update, halo wait, product
// and Gram pass into trace[5 * item + 0..4] (device, int64).
KLS_API int kls_dcgs2_fused_step_traced(const KlsStepPlan* plan, int32_t j, const double* w,
                                        double* w_out, const double* aw, double* aw_out,
                                        int32_t slot, int64_t* trace) {
  return fused_step(plan, j, w, w_out, aw, aw_out, slot, trace);
}

// Non-zero when a fused step timed out waiting for a halo (the stream's
// error word; cleared by the read).  Synchronizes the stream.
KLS_API int kls_dcgs2_fused_error(void* stream) {
  using namespace fused;
  int dev = 0;
  cudaGetDevice(&dev);
  int* e = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto itr = g_flags.find({dev, stream});
    if (itr == g_flags.end()) return 0;
    e = itr->second.err;
  }
  int h = 0;
  cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  cudaMemcpy(&h, e, sizeof(int), cudaMemcpyDeviceToHost);
  if (h) cudaMemset(e, 0, sizeof(int));
  return h;
}
