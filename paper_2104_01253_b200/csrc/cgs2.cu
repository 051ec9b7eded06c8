// K4: the CGS2 comparator's fused "update, then project" pass
// (Cgs2State.push, ortho.py:148-151): w = v - Q s followed by c = Q^T w —
// the reference's MvTimesMatAddMv + MvTransMv pair — in one launch that
// reads Q from HBM once.  So CGS2 costs three passes over Q per column (the
// first projection, this, and the final update with its fused norm) instead
// of four: an equally tuned baseline for DCGS2's two.
//
// Default (k <= 256): project_gram_reg_kernel keeps each warp's share of a
// row chunk of Q in registers between the two looks (below).  For k > 256
// and for ragged tails, project_gram_kernel re-reads a 512-row chunk through
// L2, the first look marked evict_last and the second evict_first.
//
// Measured alternatives: staging the chunk's whole panel in
// shared memory by cp.async.bulk caps the chunk at 64-128 rows for k >= 100
// (two stages in 227 KB), and bulk copies that small run at 2.4-4.5 TB/s;
// splitting the panel across a thread-block cluster (DSMEM exchange of the
// partial Q s) restores 2 KB copies but the per-chunk cluster handshake
// starves a two-stage pipeline (< 2.7 TB/s).
#include "gram.cuh"

#include <cstdlib>
#include <cstring>

namespace {

using namespace kls;
using namespace kls::gram;

constexpr int kPRP = 1;        // row pairs per lane: 8 warps x 64 rows = 512-row chunks
constexpr int kPBlocks = 3;    // CTAs per SM
constexpr int kPVirt = 148;    // virtual CTAs per segment (a third of the grid)

template <int NC>
struct PgPack {
  double v[NC > 0 ? NC : 1];
};


// L2 cache-policy loads for the LDG variant: the first look at a chunk's Q
// rows marks them evict_last so the second look (evict_first) hits in L2.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double2 ld_pair_policy(const double* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
template <bool CHECK>
__device__ __forceinline__ double2 load_pair_pol(const double* col, int64_t r, int64_t m,
                                                 uint64_t pol) {
  if (!CHECK || r + 1 < m) return ld_pair_policy(col + r, pol);
  double2 v = make_double2(0.0, 0.0);
  if (r < m) v.x = col[r];
  return v;
}

// Operands of one segment (pointers offset to its first row).
struct PgRows {
  const double* Q;
  int64_t ldq;
  int32_t k;
  int64_t m;  // the segment's rows
};

template <bool CHECK>
__device__ __forceinline__ void pg_chunk(const PgRows& p, double* v, const double* ss,
                                         int64_t wbase, int lane, double* wacc, double& xn) {
  constexpr int RP = kPRP;
  const uint64_t keep = policy_evict_last();
  const uint64_t drop = policy_evict_first();
  double2 acc[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) acc[r] = make_double2(0.0, 0.0);
  const int ng = (p.k + kG - 1) / kG;
  // first look: 8 columns in flight per lane (HBM latency), marked evict_last
  constexpr int kA = 2 * kG;
  for (int c0 = 0; c0 < p.k; c0 += kA) {
    double2 q[kA][RP];
#pragma unroll
    for (int cc = 0; cc < kA; ++cc) {
      const int c = c0 + cc;
      const double* col = p.Q + static_cast<int64_t>(c < p.k ? c : 0) * p.ldq;
#pragma unroll
      for (int r = 0; r < RP; ++r)
        q[cc][r] = c < p.k ? load_pair_pol<CHECK>(col, wbase + 64 * r + 2 * lane, p.m, keep)
                           : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int cc = 0; cc < kA; ++cc) {
      const double s = c0 + cc < p.k ? ss[c0 + cc] : 0.0;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        acc[r].x = fma(q[cc][r].x, s, acc[r].x);
        acc[r].y = fma(q[cc][r].y, s, acc[r].y);
      }
    }
  }
  double2 w[RP];
#pragma unroll
  for (int r = 0; r < RP; ++r) {
    const int64_t row = wbase + 64 * r + 2 * lane;
    const double2 a = load_pair_rw<CHECK>(v, row, p.m);
    w[r].x = a.x + -1.0 * acc[r].x;
    w[r].y = a.y + -1.0 * acc[r].y;
    store_pair<CHECK>(v, row, p.m, w[r]);
    if (CHECK) {
      if (row >= p.m) w[r].x = 0.0;
      if (row + 1 >= p.m) w[r].y = 0.0;
    }
    xn = fma(w[r].x, w[r].x, xn);
    xn = fma(w[r].y, w[r].y, xn);
  }
  // second look at the chunk's Q rows (L2): c += Q^T w
  for (int g = 0; g < ng; ++g) {
    double2 q[kG][RP];
#pragma unroll
    for (int cc = 0; cc < kG; ++cc) {
      const int c = g * kG + cc;
      const double* col = p.Q + static_cast<int64_t>(c < p.k ? c : 0) * p.ldq;
#pragma unroll
      for (int r = 0; r < RP; ++r)
        q[cc][r] = c < p.k ? load_pair_pol<CHECK>(col, wbase + 64 * r + 2 * lane, p.m, drop)
                           : make_double2(0.0, 0.0);
    }
    double a[kG];
#pragma unroll
    for (int cc = 0; cc < kG; ++cc) {
      a[cc] = 0.0;
#pragma unroll
      for (int r = 0; r < RP; ++r) {
        a[cc] = fma(q[cc][r].x, w[r].x, a[cc]);
        a[cc] = fma(q[cc][r].y, w[r].y, a[cc]);
      }
    }
    const double sred = warp_transpose_reduce<kG>(a, lane);
    if ((lane & (32 / kG - 1)) == 0) wacc[g * kG + warp_slot<kG>(lane)] += sred;
  }
}

// Launch arguments shared by both variants.
struct PgArgs {
  const double* Q;
  int64_t ldq;
  int32_t k;
  int32_t xnorm;
  seg::Plan P;
  seg::Ws ws;
  seg::Dest d;
};

// Item epilogue of both variants: the 8 warps' accumulators (sacc rows,
// stride) and xn in warp order -> the item partial (plain stores).
__device__ __forceinline__ void pg_store(const PgArgs& a, int it, const double* sacc, int stride,
                                         double xn) {
  __shared__ double sx[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double t = warp_sum(xn);
  if (lane == 0) sx[warp] = t;
  __syncthreads();
  const int nv = a.k + (a.xnorm ? 1 : 0);
  seg::item_store<kThreads>(a.ws, it, nv, threadIdx.x, [&](int i) {
    double r = 0.0;
    if (i < a.k) {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) r += sacc[w * stride + i];
    } else {
#pragma unroll
      for (int w = 0; w < kWarps; ++w) r += sx[w];
    }
    return r;
  });
  __syncthreads();  // sacc / sx are read: the next item may reset them
}

template <int NC>
__global__ void __launch_bounds__(kThreads, kPBlocks)
    project_gram_kernel(PgArgs a, double* v, const double* s_dev,
                        const __grid_constant__ PgPack<NC> pk) {
  extern __shared__ double sm[];
  __shared__ double s_red[kThreads];
  __shared__ int s_flag, s_ok;
  const int ng = (a.k + kG - 1) / kG;
  const int stride = ng * kG;
  double* ss = sm;                  // coefficients, zero-padded to ng * kG
  double* sacc = sm + stride;       // [kWarps][stride]
  const double* s = NC > 0 ? pk.v : s_dev;
  for (int i = threadIdx.x; i < stride; i += kThreads) ss[i] = i < a.k ? s[i] : 0.0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* wacc = sacc + warp * stride;
  constexpr int64_t WROWS = 64 * kPRP;
  constexpr int64_t CROWS = WROWS * kWarps;
  for (int it = blockIdx.x; it < a.P.nitems; it += gridDim.x) {
    int sg, vi, V;
    seg::item_of(a.P, it, sg, vi, V);
    const int64_t base = a.P.L.off[sg];
    const PgRows pr{a.Q + base, a.ldq, a.k, a.P.L.off[sg + 1] - base};
    double* vs = v + base;
    for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
    __syncthreads();
    double xn = 0.0;
    const int64_t nchunks = (pr.m + CROWS - 1) / CROWS;
    for (int64_t ch = vi; ch < nchunks; ch += V) {
      const int64_t cbase = ch * CROWS;
      const int64_t wbase = cbase + warp * WROWS;
      if (cbase + CROWS <= pr.m)
        pg_chunk<false>(pr, vs, ss, wbase, lane, wacc, xn);
      else
        pg_chunk<true>(pr, vs, ss, wbase, lane, wacc, xn);
    }
    pg_store(a, it, sacc, stride, xn);
  }
  const int nv = a.k + (a.xnorm ? 1 : 0);
  if (seg::finish_items<kThreads, 0>(a.P, a.ws, nv, threadIdx.x, s_red, &s_flag))
    seg::seg_final<kThreads, 0>(a.P.L, a.ws, nv, a.d, threadIdx.x, &s_ok,
                                [](int o) { return (int64_t)o; });
}

template <int NC>
int launch_pg(PgArgs a, double* v, const double* s, bool host, size_t ws_bytes, cudaStream_t st) {
  PgPack<NC> pk;
  if (NC > 0) std::memcpy(pk.v, s, sizeof(double) * a.k);
  constexpr int64_t CROWS = 64 * kPRP * kWarps;
  seg::make_plan(a.P.L, CROWS, kPVirt, a.P);
  const int nv = a.k + (a.xnorm ? 1 : 0);
  if (seg::plan_ws_bytes(a.P, nv) > ws_bytes) return fail(KLS_ENOSPC, "project_gram: workspace too small");
  a.ws = seg::ws_of(a.ws.tick, a.P.nitems, nv);
  const int grid = std::max(1, std::min(a.P.nitems, kPBlocks * sm_count()));
  const int ng = (a.k + kG - 1) / kG;
  const size_t smem = sizeof(double) * static_cast<size_t>(ng * kG) * (1 + kWarps);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(project_gram_kernel<NC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "project_gram smem: %s", cudaGetErrorString(e));
  }
  project_gram_kernel<NC><<<grid, kThreads, smem, st>>>(a, v, host ? nullptr : s, pk);
  return check_launch("project_gram_kernel");
}

// ---------------------------------------------------------------------------
// Register-resident variant (default for k <= 256): Q crosses HBM once and
// is never re-read.  A virtual CTA takes row chunks of R = 64 * RB rows of
// its segment; consumer warp w owns the columns w, w + 8, ... (CPW of them)
// and holds its CPW x RB row pairs of the chunk in registers.  Phase A forms
// its partial Q s per row; the 8 partials are combined in fixed warp order
// through shared memory into w = v - Q s (written back over v); phase B
// takes q_c . w from the same registers, accumulating per lane across the
// item's chunks (one cross-lane reduction per item).  CPW * RB = 16 row
// pairs (or 32 at CPW = 32) keep 16-32 KB of loads in flight per CTA; the
// window between the two looks at Q is a register file, not a cache.

constexpr int kRegMaxK = 32 * kWarps;

template <int CPW, int RB, int NC>
__global__ void __launch_bounds__(kThreads, CPW >= 32 ? 1 : 2)
    project_gram_reg_kernel(PgArgs a, double* v, const double* s_dev,
                            const __grid_constant__ PgPack<NC> pk) {
  constexpr int R = 64 * RB;
  extern __shared__ __align__(16) double rsm[];
  __shared__ double s_red[kThreads];
  __shared__ int s_flag, s_ok;
  const int k = a.k;
  const int stride = (k + kG - 1) / kG * kG;
  constexpr int kSs = CPW * kWarps;                // >= stride
  double* ss = rsm;                                // coefficients, zero-padded to kSs
  double* sacc = ss + kSs;                         // [kWarps][stride]
  double* part = sacc + kWarps * stride;           // [kWarps][R]
  double* wbuf = part + kWarps * R;                // [R]
  const double* s = NC > 0 ? pk.v : s_dev;
  for (int i = threadIdx.x; i < kSs; i += kThreads) ss[i] = i < k ? s[i] : 0.0;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* mypart = part + warp * R;
  double* wacc = sacc + warp * stride;
  for (int it = blockIdx.x; it < a.P.nitems; it += gridDim.x) {
    int sg, vi, V;
    seg::item_of(a.P, it, sg, vi, V);
    const int64_t base = a.P.L.off[sg];
    const int64_t rows = a.P.L.off[sg + 1] - base;
    const double* Q = a.Q + base;
    double* vs = v + base;
    for (int i = lane; i < stride; i += 32) wacc[i] = 0.0;
    __syncthreads();
    double acc[CPW];
#pragma unroll
    for (int i = 0; i < CPW; ++i) acc[i] = 0.0;
    double xn = 0.0;
    const int64_t nfull = rows / R;
    for (int64_t ch = vi; ch < nfull; ch += V) {
      const int64_t cb = ch * R;
      // v for the rows this thread combines, fetched early
      constexpr int NV = (R + kThreads - 1) / kThreads;
      double vv[NV];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int row = threadIdx.x + kThreads * i;
        if (row < R) vv[i] = vs[cb + row];
      }
      double2 q[CPW][RB];
#pragma unroll
      for (int i = 0; i < CPW; ++i) {
        const int col = warp + kWarps * i;
        const double* cp = Q + static_cast<int64_t>(col < k ? col : 0) * a.ldq + cb + 2 * lane;
#pragma unroll
        for (int b = 0; b < RB; ++b)
          q[i][b] = col < k ? ld_stream2(cp + 64 * b) : make_double2(0.0, 0.0);
      }
      // phase A
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        double2 av = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
          const double sc = ss[warp + kWarps * i];  // zero past k (padded)
          av.x = fma(q[i][b].x, sc, av.x);
          av.y = fma(q[i][b].y, sc, av.y);
        }
        *reinterpret_cast<double2*>(mypart + 64 * b + 2 * lane) = av;
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int row = threadIdx.x + kThreads * i;
        if (row < R) {
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < kWarps; ++w) t += part[w * R + row];
          const double wv = vv[i] + -1.0 * t;
          wbuf[row] = wv;
          vs[cb + row] = wv;
          xn = fma(wv, wv, xn);
        }
      }
      __syncthreads();
      // phase B from the registers
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        const double2 wv = *reinterpret_cast<const double2*>(wbuf + 64 * b + 2 * lane);
#pragma unroll
        for (int i = 0; i < CPW; ++i) {
          acc[i] = fma(q[i][b].x, wv.x, acc[i]);
          acc[i] = fma(q[i][b].y, wv.y, acc[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CPW; ++i) {
      const int col = warp + kWarps * i;
      const double t = warp_sum(acc[i]);
      if (lane == 0 && col < k) wacc[col] = t;
    }
    __syncwarp();
    // the segment's ragged tail (< R rows) through the L2-reuse path, by the
    // virtual CTA the round-robin would give the next chunk
    if (nfull * R < rows && (nfull % V) == vi) {
      const PgRows pr{Q, a.ldq, k, rows};
      for (int64_t b0 = nfull * R; b0 < rows; b0 += 64 * kPRP * kWarps)
        pg_chunk<true>(pr, vs, ss, b0 + warp * 64 * kPRP, lane, wacc, xn);
    }
    pg_store(a, it, sacc, stride, xn);
  }
  const int nv = k + (a.xnorm ? 1 : 0);
  if (seg::finish_items<kThreads, 0>(a.P, a.ws, nv, threadIdx.x, s_red, &s_flag))
    seg::seg_final<kThreads, 0>(a.P.L, a.ws, nv, a.d, threadIdx.x, &s_ok,
                                [](int o) { return (int64_t)o; });
}

template <int CPW, int NC>
int launch_pg_reg(PgArgs a, double* v, const double* s, bool host, size_t ws_bytes,
                  cudaStream_t st) {
  constexpr int RB = CPW >= 16 ? 1 : 16 / CPW;
  constexpr int R = 64 * RB;
  constexpr int blocks = CPW >= 32 ? 1 : 2;
  PgPack<NC> pk;
  if (NC > 0) std::memcpy(pk.v, s, sizeof(double) * a.k);
  auto kern = project_gram_reg_kernel<CPW, RB, NC>;
  // virtual CTAs per segment: a third of the physical grid (so 1..8 ranks'
  // shares of the 24 segments keep every SM busy)
  seg::make_plan(a.P.L, R, blocks == 2 ? 98 : 49, a.P);
  const int nv = a.k + (a.xnorm ? 1 : 0);
  if (seg::plan_ws_bytes(a.P, nv) > ws_bytes) return fail(KLS_ENOSPC, "project_gram: workspace too small");
  a.ws = seg::ws_of(a.ws.tick, a.P.nitems, nv);
  const int grid = std::max(1, std::min(a.P.nitems, blocks * sm_count()));
  const int stride = (a.k + kG - 1) / kG * kG;
  const size_t smem = sizeof(double) * (static_cast<size_t>(CPW) * kWarps +
                                        static_cast<size_t>(stride) * kWarps +
                                        static_cast<size_t>(kWarps + 1) * R);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "project_gram smem: %s", cudaGetErrorString(e));
  }
  kern<<<grid, kThreads, smem, st>>>(a, v, host ? nullptr : s, pk);
  return check_launch("project_gram_reg_kernel");
}

template <int NC>
int launch_pg_reg_cols(PgArgs a, double* v, const double* s, bool host, size_t ws_bytes,
                       cudaStream_t st) {
  const int cpw = (a.k + kWarps - 1) / kWarps;
  if (cpw <= 1) return launch_pg_reg<1, NC>(a, v, s, host, ws_bytes, st);
  if (cpw <= 2) return launch_pg_reg<2, NC>(a, v, s, host, ws_bytes, st);
  if (cpw <= 4) return launch_pg_reg<4, NC>(a, v, s, host, ws_bytes, st);
  if (cpw <= 8) return launch_pg_reg<8, NC>(a, v, s, host, ws_bytes, st);
  if (cpw <= 16) return launch_pg_reg<16, NC>(a, v, s, host, ws_bytes, st);
  return launch_pg_reg<32, NC>(a, v, s, host, ws_bytes, st);
}

}  // namespace

// w = v - Q(:, 0:k) s (written over v), then out[0:k] = Q^T w and, when
// xnorm != 0, out[k] = w.w — Cgs2State.push's first update and second
// projection (ortho.py:149-151) in one launch (1 <= k <= 2048).  s is a host
// array (carried in the launch) when s_on_host != 0, else a device array.
// Reduced over the fixed segment tree (seg.cuh); with world > 1 out receives
// the exported nodes (xstride k + xnorm).
KLS_API int kls_project_gram(const double* Q, int64_t ldq, int64_t m, int32_t k, double* v,
                             const double* s, int32_t s_on_host, int32_t xnorm, double* out,
                             const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream) {
  if ((m > 0 && (Q == nullptr || v == nullptr)) || s == nullptr || out == nullptr ||
      ws == nullptr || m < 0 ||
      k < 1 || k > 2048 || ldq < m || (ldq & 1) ||
      ((reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(v)) & 15))
    return fail(KLS_EINVAL, "project_gram: bad arguments (k=%d, 1 <= k <= 2048)", k);
  PgArgs a;
  std::memset(&a, 0, sizeof(a));
  int rc = seg::make_layout(segs, m, a.P.L);
  if (rc) return rc;
  a.Q = Q;
  a.ldq = ldq;
  a.k = k;
  a.xnorm = xnorm;
  a.ws = seg::ws_of(ws, 0, 0);
  a.d.out = out;
  a.d.xstride = k + (xnorm ? 1 : 0);
  a.d.peers.world = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k <= kRegMaxK) {
    if (!s_on_host) return launch_pg_reg_cols<0>(a, v, s, false, ws_bytes, st);
    return launch_pg_reg_cols<kRegMaxK>(a, v, s, true, ws_bytes, st);
  }
  if (!s_on_host) return launch_pg<0>(a, v, s, false, ws_bytes, st);
  if (k <= 512) return launch_pg<512>(a, v, s, true, ws_bytes, st);
  if (k <= 1024) return launch_pg<1024>(a, v, s, true, ws_bytes, st);
  return launch_pg<2048>(a, v, s, true, ws_bytes, st);
}
