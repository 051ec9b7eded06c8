// Rank-count-independent reductions.
//
// Every reduction on the path (the DCGS2 step's fused Gram, CGS2's
// projections, the flush norms, GMRES's residual norms) is summed over a
// FIXED global tree whose shape does not depend on how many ranks hold the
// rows, so 1, 2, 3, 4, 6 and 8 GPUs produce bitwise-identical scalars (and
// therefore identical H, V, GMRES iterations and Krylov-Schur locks).
//
//   * The global rows are cut into kG = 24 segments at multiples of a
//     partition unit (64 rows; a stencil's x-plane).  Rank r of N owns the
//     segments [r*24/N, (r+1)*24/N) -- the row partition itself follows the
//     segments (runtime.seg_range), so rank boundaries are segment
//     boundaries.
//   * A segment is reduced as if it were its own launch: V(s) "virtual CTAs"
//     (a function of the segment's row count only) walk it with the kernel's
//     usual schedule, each giving an item partial; the segment value is the
//     fixed-order sum of its V item partials.  Physical CTAs take items
//     round-robin, so the physical grid and the rank's other segments never
//     touch a segment's arithmetic.
//   * Segment values are combined by a fixed tree: 8 groups of 3 segments
//     ((a + b) + c), then a balanced binary tree over the 8 groups.  A rank
//     evaluates every node whose leaves it owns and exports the maximal ones
//     (exactly one node -- its subtree root -- when N divides 8); after the
//     exchange every rank evaluates the missing upper nodes from the
//     exported ones.  Each node is always the same IEEE sum of the same two
//     or three values, wherever it is evaluated.
#pragma once

#include "common.cuh"
#include "peer.cuh"

namespace kls {
namespace seg {

constexpr int kG = 24;          // global segments
constexpr int kNodes = 39;      // 24 leaves, 8 groups, 4 pairs, 2 quads, root
constexpr int kRoot = 38;
constexpr int kMaxExport = 8;   // nodes one rank exports (<= 4 for N <= 8)
constexpr int kTickBytes = 256; // segment tickets [kG] + done ticket
constexpr int kMaxVirt = 148;   // largest virtual grid of any segmented kernel

// ---- the static tree ------------------------------------------------------
__host__ __device__ constexpr int node_lo(int n) {
  return n < 24 ? n : n < 32 ? 3 * (n - 24) : n < 36 ? 6 * (n - 32) : n < 38 ? 12 * (n - 36) : 0;
}
__host__ __device__ constexpr int node_hi(int n) {
  return n < 24 ? n + 1 : n < 32 ? 3 * (n - 24) + 3 : n < 36 ? 6 * (n - 32) + 6
                                  : n < 38 ? 12 * (n - 36) + 12 : 24;
}
__host__ __device__ constexpr int node_parent(int n) {
  return n < 24 ? 24 + n / 3 : n < 32 ? 32 + (n - 24) / 2 : n < 36 ? 36 + (n - 32) / 2 : n < 38 ? 38 : -1;
}
__host__ __device__ constexpr int node_nchild(int n) { return n < 24 ? 0 : n < 32 ? 3 : 2; }
__host__ __device__ constexpr int node_child(int n, int c) {
  return n < 32 ? 3 * (n - 24) + c : n < 36 ? 24 + 2 * (n - 32) + c : n < 38 ? 32 + 2 * (n - 36) + c : 36 + c;
}

// first global segment of a rank
__host__ __device__ inline int seg_first(int rank, int world) { return rank * kG / world; }

__host__ __device__ inline bool node_inside(int n, int a, int b) {
  return a <= node_lo(n) && node_hi(n) <= b;
}

// The maximal complete subtrees of the leaf range [a, b), left to right.
// Returns their count (<= kMaxExport for every split used here).
__host__ __device__ inline int exports(int a, int b, int* ids) {
  int cnt = 0;
  int pos = a;
  while (pos < b && cnt < kMaxExport) {
    int node = pos;  // climb while the parent starts here and stays inside
    while (true) {
      const int p = node_parent(node);
      if (p < 0 || node_lo(p) != pos || !node_inside(p, a, b)) break;
      node = p;
    }
    ids[cnt++] = node;
    pos = node_hi(node);
  }
  return cnt;
}

// fold of an internal node's children, always in child order
__host__ __device__ inline double node_fold(int n, const double* val) {
  if (node_nchild(n) == 3) return (val[node_child(n, 0)] + val[node_child(n, 1)]) + val[node_child(n, 2)];
  return val[node_child(n, 0)] + val[node_child(n, 1)];
}

// ---- layouts --------------------------------------------------------------
struct Layout {
  int64_t off[kG + 1];  // local row offsets of the local segments; off[nseg] = m_local
  int32_t nseg;         // local segments
  int32_t gseg0;        // global index of the first local segment
  int32_t world, rank;
};

// A kernel's item plan: segment s has ibase[s+1] - ibase[s] virtual CTAs.
struct Plan {
  Layout L;
  int32_t ibase[kG + 1];
  int32_t nitems;
};

// Global row where segment k starts (k in [0, kG]).
__host__ __device__ inline int64_t seg_row(int64_t m, int64_t unit, int k) {
  const int64_t units = (m + unit - 1) / unit;
  const int64_t r = unit * (units * k / kG);
  return r < m ? r : m;
}

// Host: the layout of a rank's m_local rows (validated against the global
// description).  Returns 0 or a KLS_* error code.
int make_layout(const KlsSegs* s, int64_t m_local, Layout& L);
// Host: items with V(s) = clamp(ceil(rows / gran), 1, vmax).
void make_plan(const Layout& L, int64_t gran, int vmax, Plan& P);
// Host: the plan, workspace and destination of a simple segmented
// reduction of nv values over m_local rows (virtual CTAs of `gran` rows, at
// most kNormVirt per segment); out gets the results (or the exports).
constexpr int kNormVirt = 148;
struct SimpleArgs;
int make_plan_simple(const KlsSegs* s, int64_t m_local, int64_t gran, SimpleArgs& a, void* ws,
                     size_t ws_bytes, int nv, double* out);
// Host: workspace bytes for a plan reducing nv values per item.
inline size_t plan_ws_bytes(const Plan& P, int nv) {
  return kTickBytes + sizeof(double) * (static_cast<size_t>(P.nitems) + kG) * nv;
}

// ---- device pieces --------------------------------------------------------
struct Ws {
  unsigned int* tick;  // [kG] segment tickets, [kG] done ticket
  double* part;        // [nitems][nv]
  double* segv;        // [kG][nv]
};
__host__ __device__ inline Ws ws_of(void* ws, int nitems, int nv) {
  Ws w;
  w.tick = static_cast<unsigned int*>(ws);
  w.part = reinterpret_cast<double*>(static_cast<char*>(ws) + kTickBytes);
  w.segv = w.part + static_cast<size_t>(nitems) * nv;
  return w;
}

// Where results go.  world == 1: out[dst(o)] = value.  world > 1 and
// peers.world > 1: fused one-shot exchange over NVLink, then out[dst(o)].
// world > 1 without peers: this rank's exported node values,
// out[e * xstride + dst(o)] for its e-th exported node (combined later by
// kls_peer_seg_combine or kls_seg_combine).
struct Dest {
  double* out;
  int64_t xstride;
  peer::Peers peers;
  uint64_t epoch;
  int* err;
};

__device__ __forceinline__ void item_of(const Plan& P, int it, int& s, int& v, int& V) {
  s = 0;
  while (P.ibase[s + 1] <= it) ++s;
  v = it - P.ibase[s];
  V = P.ibase[s + 1] - P.ibase[s];
}

// Barrier over the NT threads of group BAR (0: the whole CTA).
template <int NT, int BAR>
__device__ __forceinline__ void gsync() {
  if (BAR == 0)
    __syncthreads();
  else
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
}

// Fixed-order sum over nb partial rows (row stride nv) of every entry by one
// thread group (sum_partials_block's order, for a group of NT threads).
template <int NT, int BAR, typename Emit>
__device__ __forceinline__ void group_sum_partials(const double* partials, int nb, int nv, int tid,
                                                   double* s_red, Emit emit) {
  int S = nv > 0 ? NT / nv : 1;
  S = S >= 16 ? 16 : S >= 8 ? 8 : S >= 4 ? 4 : S >= 2 ? 2 : 1;
  const int per_round = NT / S;
  const int slot = tid / S;
  const int sl = tid % S;
  for (int base = 0; base < nv; base += per_round) {
    const int i = base + slot;
    const bool live = slot < per_round && i < nv;
    double v = 0.0;
    if (live) {
      double a[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int b = sl;
      for (; b + 7 * S < nb; b += 8 * S) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] += __ldcg(partials + static_cast<int64_t>(b + u * S) * nv + i);
      }
      for (; b < nb; b += S) a[0] += __ldcg(partials + static_cast<int64_t>(b) * nv + i);
      v = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    }
    s_red[tid] = v;
    gsync<NT, BAR>();
    if (live && sl == 0) {
      double t = 0.0;
      for (int k = 0; k < S; ++k) t += s_red[tid + k];
      emit(i, t);
    }
    gsync<NT, BAR>();
  }
}

// Store one item's nv values (get(i)) to its partial row: plain stores,
// nothing waits (the fence and the segment tickets come once per CTA, in
// finish_items).  The group must have finished the item's accumulation.
template <int NT, typename Get>
__device__ __forceinline__ void item_store(Ws ws, int it, int nv, int tid, Get get) {
  double* part = ws.part + static_cast<int64_t>(it) * nv;
  for (int i = tid; i < nv; i += NT) part[i] = get(i);
}

// Once per CTA after its last item: publish the CTA's item partials
// (fence), take the segment tickets for the items it processed (items
// blockIdx.x, + gridDim.x, ...), reduce every segment this CTA completed
// (its V item partials in fixed order, group_sum_partials), and count
// completed segments.  Returns true in the group of the CTA that completed
// the LAST segment (it then runs seg_final).  s_red: NT doubles of shared
// memory; s_flag: one shared int.
template <int NT, int BAR>
__device__ __forceinline__ bool finish_items(const Plan& P, Ws ws, int nv, int tid, double* s_red,
                                             int* s_flag) {
  __shared__ int s_seg[kG], s_cnt[kG], s_done[kG], s_nt;
  __threadfence();
  gsync<NT, BAR>();
  if (tid == 0) {  // the segments this CTA's items belong to, with item counts
    int n = 0;
    for (int it = blockIdx.x; it < P.nitems; it += gridDim.x) {
      int s = 0;
      while (P.ibase[s + 1] <= it) ++s;
      if (n == 0 || s_seg[n - 1] != s) {
        s_seg[n] = s;
        s_cnt[n] = 0;
        ++n;
      }
      ++s_cnt[n - 1];
    }
    s_nt = n;
  }
  gsync<NT, BAR>();
  const int nt = s_nt;
  if (tid < nt) {  // all tickets at once: one round trip
    const int s = s_seg[tid];
    const unsigned V = static_cast<unsigned>(P.ibase[s + 1] - P.ibase[s]);
    s_done[tid] = atomicAdd(ws.tick + s, static_cast<unsigned>(s_cnt[tid])) + s_cnt[tid] == V;
  }
  gsync<NT, BAR>();
  int completed = 0;
  for (int k = 0; k < nt; ++k) {
    if (!s_done[k]) continue;
    const int s = s_seg[k];
    const int V = P.ibase[s + 1] - P.ibase[s];
    __threadfence();
    double* sv = ws.segv + static_cast<int64_t>(s) * nv;
    group_sum_partials<NT, BAR>(ws.part + static_cast<int64_t>(P.ibase[s]) * nv, V, nv, tid,
                                s_red, [&](int i, double t) { sv[i] = t; });
    if (tid == 0) ws.tick[s] = 0u;
    ++completed;
  }
  if (completed == 0) return false;
  __threadfence();
  gsync<NT, BAR>();
  if (tid == 0) {
    const unsigned c = static_cast<unsigned>(completed);
    const bool last = atomicAdd(ws.tick + kG, c) + c == static_cast<unsigned>(P.L.nseg);
    if (last) ws.tick[kG] = 0u;
    *s_flag = last ? 1 : 0;
  }
  gsync<NT, BAR>();
  const bool fin = *s_flag != 0;
  if (fin) __threadfence();
  return fin;
}

// Local tree of one output: val[] gets every node whose leaves this rank
// owns, from the local segment values segv[(leaf - gseg0) * stride + o].
__device__ __forceinline__ void local_tree(const Layout& L, const double* segv, int64_t stride,
                                           int o, double* val) {
  const int a = L.gseg0, b = L.gseg0 + L.nseg;
  for (int l = a; l < b; ++l) val[l] = __ldcg(segv + static_cast<int64_t>(l - a) * stride + o);
  for (int n = kG; n < kNodes; ++n)
    if (node_inside(n, a, b)) val[n] = node_fold(n, val);
}

// The same from leaf values given by leaf(s) for local segment s.
template <typename Leaf>
__device__ __forceinline__ void local_tree_from(const Layout& L, Leaf leaf, double* val) {
  const int a = L.gseg0, b = L.gseg0 + L.nseg;
  for (int l = a; l < b; ++l) val[l] = leaf(l - a);
  for (int n = kG; n < kNodes; ++n)
    if (node_inside(n, a, b)) val[n] = node_fold(n, val);
}

// The whole tree of one rank holding all 24 segments, straight-line (the
// same folds as local_tree + combine: 8 groups of 3, then pairs, quads,
// root), so the 24 leaf loads are independent.
template <typename Leaf>
__device__ __forceinline__ double root24(Leaf leaf) {
  double g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) g[i] = (leaf(3 * i) + leaf(3 * i + 1)) + leaf(3 * i + 2);
  const double p0 = g[0] + g[1], p1 = g[2] + g[3], p2 = g[4] + g[5], p3 = g[6] + g[7];
  return (p0 + p1) + (p2 + p3);
}

// Combine: val[] holds every rank's exported nodes (have[] marks them);
// the missing upper nodes are folded; returns the root.
__device__ __forceinline__ double combine_tree(double* val, bool* have) {
  for (int n = kG; n < kNodes; ++n) {
    if (have[n]) continue;
    bool ready = true;
    for (int c = 0; c < node_nchild(n); ++c) ready = ready && have[node_child(n, c)];
    if (ready) {  // nodes below an exported one stay unevaluated
      val[n] = node_fold(n, val);
      have[n] = true;
    }
  }
  return val[kRoot];
}

// The one-shot flag exchange of the fused path (one thread per peer).
// Returns false on a timeout (err set, outputs poisoned by the caller).
template <int NT, int BAR>
__device__ __forceinline__ bool peer_exchange(const Dest& d, int tid, int* s_ok) {
  if (tid == 0) *s_ok = 1;
  gsync<NT, BAR>();
  if (tid < d.peers.world) {
    __threadfence_system();
    peer::st_release_sys(peer::ar_flags(d.peers.buf[tid]) + d.peers.rank, d.epoch);
    if (!peer::wait_flag(peer::ar_flags(d.peers.buf[d.peers.rank]) + tid, d.epoch)) atomicExch(s_ok, 0);
  }
  gsync<NT, BAR>();
  return *s_ok != 0;
}

// Cross-rank combine of nv outputs from the exported blocks in every
// rank's peer slot (layout [e][nv]); emit(o, value).
template <int NT, typename Emit>
__device__ __forceinline__ void combine_from_slots(const Dest& d, int nv, int tid, Emit emit) {
  const int W = d.peers.world;
  if (W == 2 || W == 4 || W == 8) {
    // each rank exports exactly its subtree root (a node of the binary part
    // of the tree): all W remote loads in flight at once, then the balanced
    // tree over them in rank order -- the same folds as combine_tree
    for (int o = tid; o < nv; o += NT) {
      double v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        if (r < W) v[r] = *(reinterpret_cast<const volatile double*>(
                              peer::slot(d.peers.buf[r], d.peers.cap, d.epoch)) + o);
      if (W == 8) {
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] = v[2 * r] + v[2 * r + 1];
      }
      if (W >= 4) {
        v[0] = v[0] + v[1];
        v[1] = v[2] + v[3];
      }
      emit(o, v[0] + v[1]);
    }
    return;
  }
  for (int o = tid; o < nv; o += NT) {
    double val[kNodes];
    bool have[kNodes];
#pragma unroll 1
    for (int n = 0; n < kNodes; ++n) have[n] = false;
#pragma unroll 1
    for (int r = 0; r < d.peers.world; ++r) {
      int ids[kMaxExport];
      const int ne = exports(seg_first(r, d.peers.world), seg_first(r + 1, d.peers.world), ids);
      const volatile double* sl = peer::slot(d.peers.buf[r], d.peers.cap, d.epoch);
      for (int e = 0; e < ne; ++e) {
        val[ids[e]] = sl[static_cast<int64_t>(e) * nv + o];
        have[ids[e]] = true;
      }
    }
    emit(o, combine_tree(val, have));
  }
}

// Final stage, run by the group that completed the last segment: local
// tree per output, then (world 1) the root, (fused peers) the exchange and
// combine, or (otherwise) the exported node values.  dst(o) maps an output
// to its position in `out`.  Returns false when the peer exchange failed.
template <int NT, int BAR, typename Dst>
__device__ __forceinline__ bool seg_final(const Layout& L, Ws ws, int nv, const Dest& d, int tid,
                                          int* s_ok, Dst dst) {
  int ids[kMaxExport];
  const int ne = exports(L.gseg0, L.gseg0 + L.nseg, ids);
  const bool fused = L.world > 1 && d.peers.world > 1;
  double* mine = fused ? peer::slot(d.peers.buf[d.peers.rank], d.peers.cap, d.epoch) : nullptr;
  for (int o = tid; o < nv; o += NT) {
    if (L.world == 1) {
      d.out[dst(o)] = root24([&](int l) { return __ldcg(ws.segv + static_cast<int64_t>(l) * nv + o); });
      continue;
    }
    double val[kNodes];
    local_tree(L, ws.segv, nv, o, val);
    if (fused) {
      for (int e = 0; e < ne; ++e) mine[static_cast<int64_t>(e) * nv + o] = val[ids[e]];
    } else {
      for (int e = 0; e < ne; ++e) d.out[static_cast<int64_t>(e) * d.xstride + dst(o)] = val[ids[e]];
    }
  }
  if (!fused) return true;
  if (!peer_exchange<NT, BAR>(d, tid, s_ok)) {
    if (tid == 0) *d.err = 1;
    for (int o = tid; o < nv; o += NT) d.out[dst(o)] = __longlong_as_double(0x7ff8000000000000ll);
    return false;
  }
  combine_from_slots<NT>(d, nv, tid, [&](int o, double v) { d.out[dst(o)] = v; });
  return true;
}

// CTA sum of NV per-thread values (warp butterflies, warps in index order)
// into sv[NV] (shared); every thread must call it.
template <int NV>
__device__ __forceinline__ void block_sum(const double (&v)[NV], double* sv) {
  __shared__ double sred[32][NV];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const double s = warp_sum(v[i]);
    if (lane == 0) sred[warp][i] = s;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += sred[w][threadIdx.x];
    sv[threadIdx.x] = s;
  }
  __syncthreads();
}

// Launch arguments of the simple segmented reductions (norms).
struct SimpleArgs {
  Plan P;
  Ws ws;
  Dest d;
};

// Item loop of a simple segmented reduction of NV per-thread accumulators
// (blockDim.x == NT): body(row0, rows, v, V, acc) accumulates this thread's
// share of an item's rows (virtual CTA v of V over rows [row0, row0 +
// rows)); the outputs are o = 0..NV-1 at out[o] (exports at
// out[e * xstride + o]).
template <int NT, int NV, typename Body>
__device__ __forceinline__ void run_simple(const SimpleArgs& A, Body body) {
  __shared__ double s_red[NT];
  __shared__ double sv[NV];
  __shared__ int s_flag, s_ok;
  for (int it = blockIdx.x; it < A.P.nitems; it += gridDim.x) {
    int s, v, V;
    item_of(A.P, it, s, v, V);
    const int64_t r0 = A.P.L.off[s];
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
    body(r0, A.P.L.off[s + 1] - r0, v, V, acc);
    block_sum<NV>(acc, sv);
    item_store<NT>(A.ws, it, NV, threadIdx.x, [&](int i) { return sv[i]; });
  }
  if (finish_items<NT, 0>(A.P, A.ws, NV, threadIdx.x, s_red, &s_flag))
    seg_final<NT, 0>(A.P.L, A.ws, NV, A.d, threadIdx.x, &s_ok, [](int o) { return (int64_t)o; });
}

}  // namespace seg
}  // namespace kls
