// Host side of the rank-count-independent reductions (seg.cuh): segment
// layouts and item plans, and the cross-rank combine for the paths that
// exchange exported nodes outside a kernel (NCCL all_gather, unfused peer
// exchange).
#include "seg.cuh"

namespace kls {
namespace seg {

namespace cache {
// The last layouts / plans built on this thread: a DCGS2 step asks for the
// same ones every launch, and building them costs ~50 64-bit divisions
// (~1.5 us of host time per launch at config 1's 20 us step).
struct LayoutKey {
  int64_t m, unit, m_local;
  int32_t world, rank;
  bool operator==(const LayoutKey& o) const {
    return m == o.m && unit == o.unit && m_local == o.m_local && world == o.world &&
           rank == o.rank;
  }
};
constexpr int kCache = 4;
thread_local LayoutKey t_lkey[kCache];
thread_local Layout t_lval[kCache];
thread_local int t_lnext = 0, t_lfill = 0;

struct PlanKey {
  LayoutKey l;
  int64_t gran;
  int vmax;
  bool operator==(const PlanKey& o) const { return l == o.l && gran == o.gran && vmax == o.vmax; }
};
thread_local PlanKey t_pkey[kCache];
thread_local Plan t_pval[kCache];
thread_local int t_pnext = 0, t_pfill = 0;

}  // namespace cache
using namespace cache;

static int make_layout_uncached(const KlsSegs* s, int64_t m_local, Layout& L);

int make_layout(const KlsSegs* s, int64_t m_local, Layout& L) {
  const LayoutKey k{s ? s->m : -1, s ? s->unit : -1, m_local, s ? s->world : -1, s ? s->rank : -1};
  for (int i = 0; i < t_lfill; ++i)
    if (t_lkey[i] == k) {
      L = t_lval[i];
      return KLS_OK;
    }
  const int rc = make_layout_uncached(s, m_local, L);
  if (rc) return rc;
  t_lkey[t_lnext] = k;
  t_lval[t_lnext] = L;
  t_lnext = (t_lnext + 1) % kCache;
  if (t_lfill < kCache) ++t_lfill;
  return KLS_OK;
}

static int make_layout_uncached(const KlsSegs* s, int64_t m_local, Layout& L) {
  KlsSegs d;
  if (s == nullptr) {
    d.m = m_local;
    d.unit = 64;
    d.world = 1;
    d.rank = 0;
    s = &d;
  }
  if (s->world < 1 || s->world > kG || s->rank < 0 || s->rank >= s->world || s->unit < 1 ||
      s->m < 0)
    return fail(KLS_EINVAL, "segments: bad layout (m=%lld unit=%lld world=%d rank=%d)",
                (long long)s->m, (long long)s->unit, s->world, s->rank);
  if (s->unit & 1)
    return fail(KLS_EINVAL, "segments: the partition unit must be even (16-byte aligned segments)");
  const int a = seg_first(s->rank, s->world), b = seg_first(s->rank + 1, s->world);
  const int64_t r0 = seg_row(s->m, s->unit, a);
  if (seg_row(s->m, s->unit, b) - r0 != m_local)
    return fail(KLS_EINVAL, "segments: %lld local rows, the layout gives rank %d rows [%lld, %lld)",
                (long long)m_local, s->rank, (long long)r0, (long long)seg_row(s->m, s->unit, b));
  L.nseg = b - a;
  L.gseg0 = a;
  L.world = s->world;
  L.rank = s->rank;
  for (int i = 0; i <= kG; ++i) L.off[i] = i <= L.nseg ? seg_row(s->m, s->unit, a + i) - r0 : m_local;
  return KLS_OK;
}

static void make_plan_uncached(const Layout& L, int64_t gran, int vmax, Plan& P);

void make_plan(const Layout& L, int64_t gran, int vmax, Plan& P) {
  // the layout's identity: its local offsets are a function of these
  LayoutKey lk{L.off[L.nseg], L.gseg0, L.nseg, L.world, L.rank};
  for (int i = 0; i <= L.nseg; ++i) lk.unit = lk.unit * 1000003 + L.off[i];
  const PlanKey k{lk, gran, vmax};
  for (int i = 0; i < t_pfill; ++i)
    if (t_pkey[i] == k && t_pval[i].L.nseg == L.nseg &&
        t_pval[i].L.off[L.nseg] == L.off[L.nseg] && t_pval[i].L.gseg0 == L.gseg0) {
      P = t_pval[i];
      return;
    }
  make_plan_uncached(L, gran, vmax, P);
  t_pkey[t_pnext] = k;
  t_pval[t_pnext] = P;
  t_pnext = (t_pnext + 1) % kCache;
  if (t_pfill < kCache) ++t_pfill;
}

static void make_plan_uncached(const Layout& L, int64_t gran, int vmax, Plan& P) {
  P.L = L;
  int n = 0;
  for (int s = 0; s < kG; ++s) {
    P.ibase[s] = n;
    if (s < L.nseg) {
      const int64_t rows = L.off[s + 1] - L.off[s];
      int64_t v = (rows + gran - 1) / gran;
      v = v < 1 ? 1 : v > vmax ? vmax : v;
      n += static_cast<int>(v);
    }
  }
  P.ibase[kG] = n;
  P.nitems = n;
}

int make_plan_simple(const KlsSegs* s, int64_t m_local, int64_t gran, SimpleArgs& a, void* ws,
                     size_t ws_bytes, int nv, double* out) {
  int rc = make_layout(s, m_local, a.P.L);
  if (rc) return rc;
  make_plan(a.P.L, gran, kNormVirt, a.P);
  if (ws == nullptr || plan_ws_bytes(a.P, nv) > ws_bytes)
    return fail(KLS_ENOSPC, "segmented reduction: workspace %zu bytes < %zu needed", ws_bytes,
                plan_ws_bytes(a.P, nv));
  a.ws = ws_of(ws, a.P.nitems, nv);
  a.d.out = out;
  a.d.xstride = nv;
  a.d.peers.world = 0;
  a.d.epoch = 0;
  a.d.err = nullptr;
  return KLS_OK;
}

}  // namespace seg
}  // namespace kls

namespace {

using namespace kls;
using namespace kls::seg;

// blocks: [world][kMaxExport][stride]: rank r's exported node values (its
// e-th exported node at [r][e][o]); out[o] = the tree's root.
__global__ void __launch_bounds__(kThreads) seg_combine_kernel(const double* __restrict__ blocks,
                                                               int nout, int64_t stride,
                                                               int world, double* out) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double val[kNodes];
    bool have[kNodes];
#pragma unroll 1
    for (int n = 0; n < kNodes; ++n) have[n] = false;
#pragma unroll 1
    for (int r = 0; r < world; ++r) {
      int ids[kMaxExport];
      const int ne = exports(seg_first(r, world), seg_first(r + 1, world), ids);
      for (int e = 0; e < ne; ++e) {
        val[ids[e]] = blocks[(static_cast<int64_t>(r) * kMaxExport + e) * stride + o];
        have[ids[e]] = true;
      }
    }
    out[o] = combine_tree(val, have);
  }
}

}  // namespace

// This rank's global rows [lo, hi) under the layout.
KLS_API int kls_seg_rows(const KlsSegs* s, int64_t* lo, int64_t* hi) {
  if (s == nullptr || lo == nullptr || hi == nullptr || s->world < 1 || s->world > kG ||
      s->rank < 0 || s->rank >= s->world || s->unit < 1 || s->m < 0)
    return fail(KLS_EINVAL, "seg_rows: bad layout");
  *lo = seg_row(s->m, s->unit, seg_first(s->rank, s->world));
  *hi = seg_row(s->m, s->unit, seg_first(s->rank + 1, s->world));
  return KLS_OK;
}

// The tree nodes a rank exports (ids, left to right); returns their count.
KLS_API int kls_seg_exports(int32_t rank, int32_t world, int32_t* ids) {
  if (ids == nullptr || world < 1 || world > kG || rank < 0 || rank >= world)
    return fail(KLS_EINVAL, "seg_exports: bad rank / world");
  int tmp[kMaxExport];
  const int n = exports(seg_first(rank, world), seg_first(rank + 1, world), tmp);
  for (int i = 0; i < n; ++i) ids[i] = tmp[i];
  return n;
}

// Combine the gathered export blocks of all ranks into the global values.
KLS_API int kls_seg_combine(const double* blocks, int32_t nout, int64_t stride, int32_t world,
                            double* out, void* stream) {
  if (blocks == nullptr || out == nullptr || nout < 0 || stride < nout || world < 1 ||
      world > kG)
    return fail(KLS_EINVAL, "seg_combine: bad arguments");
  if (nout == 0) return KLS_OK;
  const int grid = static_cast<int>(std::min<int64_t>(ceil_div(nout, kThreads), 64));
  seg_combine_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(blocks, nout, stride,
                                                                               world, out);
  return check_launch("seg_combine_kernel");
}
