// K1, TMA-staged: the Q column tiles of a row chunk are brought into shared
// memory with bulk asynchronous copies (cp.async.bulk, completed on
// mbarriers) by one producer warp, while 8 consumer warps form the partial
// dots from shared memory and reduce-scatter them across each warp with a
// halving butterfly.
//
// Work is a list of items (seg.cuh): item (s, v) is virtual CTA v of the
// V(s) that walk segment s with the chunk schedule of ChunkWalk (1024-row
// chunks round-robin, the remainder split evenly).  A persistent CTA per SM
// takes items round-robin; after each item the consumer warps sum their
// per-warp accumulators in warp order into the item partial and store it
// (plain stores: nothing waits); after its last item a CTA publishes its
// partials once and takes the segment tickets, and the CTA that completes a
// segment reduces the segment's item partials (fixed order).  The CTA that completes the launch's last segment
// evaluates the fixed segment tree (and, with NVLink peers, exchanges the
// rank's exported nodes and combines them) and runs the fused DCGS2 scalar
// step.  The arithmetic of every segment depends only on its rows, so the
// result is identical for any number of ranks and any physical grid.
//
// Pipeline per CTA: a 4-stage ring of 4 columns x 1024 rows (32 KB per
// stage) for Q, and a double-buffered slot for the chunk's right-hand
// vectors; the producer streams straight across item boundaries.
#include "gram.cuh"
#include "tma.cuh"

namespace kls {
namespace gram {
namespace {

using namespace kls::tma;

constexpr int kR = 1024;          // rows per chunk
constexpr int kRPt = 2;           // row pairs per lane (8 warps x 64 x 2 = 1024)
constexpr int kStages = 4;
constexpr int kProducerWarp = kWarps;
constexpr int kConsumers = kWarps * 32;
constexpr int kTmaThreads = (kWarps + 1) * 32;
constexpr int kPanelTma = 256;    // basis columns per launch (per-warp accumulators in smem)
constexpr int64_t kAlwaysBalance = int64_t(1) << 40;  // items: always split the remainder

template <int NX>
__global__ void __launch_bounds__(kTmaThreads, 1) gram_tma_kernel(GramParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ double sx[kWarps][NX + 1];
  __shared__ double s_red[kTmaThreads];
  __shared__ int s_flag, s_ok, s_fin;
  constexpr int V = kG * NX;
  const int nxb = NX + ((p.bext != nullptr && p.bext != p.x0) ? 1 : 0);  // staged rhs columns
  // layout: [mbarriers 256 B][Q ring][x double buffer][per-warp accumulators]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + kStages;
  uint64_t* xfull = empty + kStages;
  uint64_t* xempty = xfull + 2;
  double* qring = reinterpret_cast<double*>(smem + 256);
  double* xbuf = qring + static_cast<size_t>(kStages) * kG * kR;
  double* sacc = xbuf + static_cast<size_t>(2) * 3 * kR;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ng = (p.k + kG - 1) / kG;
  const int stride = ng * V;
  const int nq = p.k * NX;
  const int has_b = p.bext != nullptr ? 1 : 0;
  const int nv = nq + has_b * NX + (p.xnorm ? 1 : 0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kWarps);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(xfull + s, 1);
      mbar_init(xempty + s, kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_fin = 0;
  }
  if (warp < kWarps) {
    double* wacc = sacc + warp * stride;
    for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
  }
  // rows past a short chunk's end are multiplied by zeroed x rows: the ring
  // must hold finite values there.  Short chunks occur in every item's
  // balanced remainder, so the ring always starts zeroed (stale rows left
  // by earlier chunks are finite basis values).
  for (int i = threadIdx.x; i < kStages * kG * kR / 2; i += blockDim.x)
    reinterpret_cast<double2*>(qring)[i] = make_double2(0.0, 0.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the bulk copies land
  __syncthreads();

  if (warp == kProducerWarp) {
    if (lane == 0) {
      uint32_t use = 0;  // Q stage fills so far
      uint32_t xuse = 0;
      int npre = 0;      // Q groups of the CTA's first chunk already in flight
      if (p.qprefetch && blockIdx.x < p.P.nitems) {
        int s, v, Vn;
        seg::item_of(p.P, blockIdx.x, s, v, Vn);
        const int64_t base = p.P.L.off[s];
        const int64_t m64 = (p.P.L.off[s + 1] - base) & ~static_cast<int64_t>(63);
        int64_t row, nr;
        ChunkWalk<kR> cw(m64, Vn, v, kAlwaysBalance);
        if (cw.next(row, nr)) {
          const uint32_t bytes = static_cast<uint32_t>(nr) * sizeof(double);
          npre = min(ng, kStages);
          for (int g = 0; g < npre; ++g, ++use) {
            const int ncols = min(kG, p.k - g * kG);
            mbar_expect_tx(full + g, static_cast<uint32_t>(ncols) * bytes);
            for (int cc = 0; cc < ncols; ++cc)
              bulk_g2s(qring + (static_cast<size_t>(g) * kG + cc) * kR,
                       p.Q + base + static_cast<int64_t>(g * kG + cc) * p.ldq + row, bytes, full + g);
          }
        }
      }
      pdl_wait();  // x vectors (and, without qprefetch, the basis) from the preceding kernels
      for (int it = blockIdx.x; it < p.P.nitems; it += gridDim.x) {
        int s, v, Vn;
        seg::item_of(p.P, it, s, v, Vn);
        const int64_t base = p.P.L.off[s];
        const int64_t m64 = (p.P.L.off[s + 1] - base) & ~static_cast<int64_t>(63);
        const double* xsrc[3] = {p.x0 + base, p.x1 != nullptr ? p.x1 + base : nullptr,
                                 p.bext != nullptr ? p.bext + base : nullptr};
        const double* qb = p.Q + base;
        int64_t row, nr;
        for (ChunkWalk<kR> cw(m64, Vn, v, kAlwaysBalance); cw.next(row, nr); ++xuse) {
          const uint32_t bytes = static_cast<uint32_t>(nr) * sizeof(double);
          const int xs = xuse & 1;
          if (xuse >= 2) mbar_wait(xempty + xs, ((xuse >> 1) - 1) & 1);
          mbar_expect_tx(xfull + xs, static_cast<uint32_t>(nxb) * bytes);
          for (int t = 0; t < nxb; ++t)
            bulk_g2s(xbuf + (static_cast<size_t>(xs) * 3 + t) * kR, xsrc[t] + row, bytes, xfull + xs);
          for (int g = npre; g < ng; ++g, ++use) {
            const int st = use % kStages;
            const uint32_t round = use / kStages;
            if (round >= 1) mbar_wait(empty + st, (round - 1) & 1);
            const int ncols = min(kG, p.k - g * kG);
            mbar_expect_tx(full + st, static_cast<uint32_t>(ncols) * bytes);
            for (int cc = 0; cc < ncols; ++cc)
              bulk_g2s(qring + (static_cast<size_t>(st) * kG + cc) * kR,
                       qb + static_cast<int64_t>(g * kG + cc) * p.ldq + row, bytes, full + st);
          }
          npre = 0;
        }
      }
    }
  } else {
    pdl_wait();  // the tail rows read x and Q directly
    double* wacc = sacc + warp * stride;
    const int64_t wrow = warp * (64 * kRPt);
    uint32_t use = 0;
    uint32_t xuse = 0;
    for (int it = blockIdx.x; it < p.P.nitems; it += gridDim.x) {
      int s, v, Vn;
      seg::item_of(p.P, it, s, v, Vn);
      const int64_t base = p.P.L.off[s];
      const int64_t rows = p.P.L.off[s + 1] - base;
      const int64_t m64 = rows & ~static_cast<int64_t>(63);
      double ex[NX];
#pragma unroll
      for (int t = 0; t < NX; ++t) ex[t] = 0.0;
      double xn = 0.0;
      int64_t row, nr;  // nr: a multiple of 64
      for (ChunkWalk<kR> cw(m64, Vn, v, kAlwaysBalance); cw.next(row, nr); ++xuse) {
        bool live[kRPt];
#pragma unroll
        for (int r = 0; r < kRPt; ++r) live[r] = wrow + 64 * r < nr;
        const int xs = xuse & 1;
        mbar_wait(xfull + xs, (xuse >> 1) & 1);
        double2 xv[NX][kRPt];
        const double* xb = xbuf + static_cast<size_t>(xs) * 3 * kR;
#pragma unroll
        for (int t = 0; t < NX; ++t)
#pragma unroll
          for (int r = 0; r < kRPt; ++r)
            xv[t][r] = live[r] ? *reinterpret_cast<const double2*>(xb + t * kR + wrow + 64 * r + 2 * lane)
                               : make_double2(0.0, 0.0);
        if (p.bext != nullptr) {
#pragma unroll
          for (int r = 0; r < kRPt; ++r) {
            const double2 b = p.bext == p.x0 || !live[r]
                                  ? xv[0][r]
                                  : *reinterpret_cast<const double2*>(xb + NX * kR + wrow + 64 * r + 2 * lane);
#pragma unroll
            for (int t = 0; t < NX; ++t) {
              ex[t] = fma(b.x, xv[t][r].x, ex[t]);
              ex[t] = fma(b.y, xv[t][r].y, ex[t]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(xempty + xs);
        if (p.xnorm) {
#pragma unroll
          for (int r = 0; r < kRPt; ++r) {
            xn = fma(xv[NX - 1][r].x, xv[NX - 1][r].x, xn);
            xn = fma(xv[NX - 1][r].y, xv[NX - 1][r].y, xn);
          }
        }
        for (int g = 0; g < ng; ++g, ++use) {
          const int st = use % kStages;
          mbar_wait(full + st, (use / kStages) & 1);
          const double* qs = qring + static_cast<size_t>(st) * kG * kR;
          double2 q[kG][kRPt];
#pragma unroll
          for (int cc = 0; cc < kG; ++cc) {
            if (g * kG + cc < p.k) {
#pragma unroll
              for (int r = 0; r < kRPt; ++r)
                q[cc][r] = *reinterpret_cast<const double2*>(qs + cc * kR + wrow + 64 * r + 2 * lane);
            } else {
#pragma unroll
              for (int r = 0; r < kRPt; ++r) q[cc][r] = make_double2(0.0, 0.0);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(empty + st);
          double acc[V];
#pragma unroll
          for (int vv = 0; vv < V; ++vv) acc[vv] = 0.0;
#pragma unroll
          for (int cc = 0; cc < kG; ++cc)
#pragma unroll
            for (int r = 0; r < kRPt; ++r)
#pragma unroll
              for (int t = 0; t < NX; ++t) {
                acc[cc * NX + t] = fma(q[cc][r].x, xv[t][r].x, acc[cc * NX + t]);
                acc[cc * NX + t] = fma(q[cc][r].y, xv[t][r].y, acc[cc * NX + t]);
              }
          const double sred = warp_transpose_reduce<V>(acc, lane);
          if ((lane & (32 / V - 1)) == 0) wacc[g * V + warp_slot<V>(lane)] += sred;
        }
      }
      // the < 64 rows past the segment's last multiple of 64: read directly
      // by the segment's last virtual CTA
      if (m64 < rows && v == Vn - 1) {
        const GramRows gr{p.Q + base, p.ldq, p.k, p.bext != nullptr ? p.bext + base : nullptr,
                          p.x0 + base, p.x1 != nullptr ? p.x1 + base : nullptr, rows, p.xnorm};
        gram_chunk<NX, kRPt, true>(gr, m64 + wrow, lane, wacc, ex, xn);
      }
      // item partial: the 8 warps' accumulators in warp order
#pragma unroll
      for (int t = 0; t < NX; ++t) {
        const double sv = warp_sum(ex[t]);
        if (lane == 0) sx[warp][t] = sv;
      }
      {
        const double sv = warp_sum(xn);
        if (lane == 0) sx[warp][NX] = sv;
      }
      seg::gsync<kConsumers, 1>();
      seg::item_store<kConsumers>(p.ws, it, nv, threadIdx.x, [&](int i) {
        double t = 0.0;
        if (i < nq) {
#pragma unroll
          for (int w = 0; w < kWarps; ++w) t += sacc[w * stride + i];
        } else if (has_b && i < nq + NX) {
#pragma unroll
          for (int w = 0; w < kWarps; ++w) t += sx[w][i - nq];
        } else {
#pragma unroll
          for (int w = 0; w < kWarps; ++w) t += sx[w][NX];
        }
        return t;
      });
      seg::gsync<kConsumers, 1>();  // every warp's accumulators are read
      for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
      __syncwarp();
    }
    if (seg::finish_items<kConsumers, 1>(p.P, p.ws, nv, threadIdx.x, s_red, &s_flag) &&
        threadIdx.x == 0)
      s_fin = 1;
  }
  // the streaming is done: a dependent update (PDL) may start staging its
  // Q tiles while the final sums and the scalar step finish here
  pdl_trigger();
  __syncthreads();
  if (!s_fin) return;
  const bool ok = seg::seg_final<kTmaThreads, 0>(p.P.L, p.ws, nv, p.d, threadIdx.x, &s_ok,
                                                  [&](int i) { return gram_dst<NX>(p, i); });
  if (ok && p.coef != nullptr) {
    __syncthreads();
    dcgs2_scalars_block(p.d.out, p.bext_row, p.qr, p.coef, p.gout);
  }
}

}  // namespace

bool tma_eligible(const GramParams& p) {
  return p.k <= kPanelTma &&
         ((reinterpret_cast<uintptr_t>(p.Q) | reinterpret_cast<uintptr_t>(p.x0) |
           reinterpret_cast<uintptr_t>(p.x1) | reinterpret_cast<uintptr_t>(p.bext)) &
          15) == 0 &&
         (p.ldq % 2) == 0;
}

template <int NX>
int launch_gram_tma(GramParams p, cudaStream_t st) {
  int grid = std::min(p.P.nitems, sm_count());
  if (grid < 1) grid = 1;
  const int ng = (p.k + kG - 1) / kG;
  const size_t smem = 256 + sizeof(double) * (static_cast<size_t>(kStages) * kG * kR + 2 * 3 * kR +
                                              static_cast<size_t>(kWarps) * ng * kG * NX);
  cudaError_t e = cudaFuncSetAttribute(gram_tma_kernel<NX>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(KLS_ECUDA, "gram_tma: smem attr: %s", cudaGetErrorString(e));
  return launch_dependent(gram_tma_kernel<NX>, dim3(grid), dim3(kTmaThreads), smem, st,
                          "gram_tma_kernel", p);
}

template int launch_gram_tma<1>(GramParams, cudaStream_t);
template int launch_gram_tma<2>(GramParams, cudaStream_t);

}  // namespace gram
}  // namespace kls
