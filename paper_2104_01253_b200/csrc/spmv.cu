// K3: operator applications y = A x (LinearOperator.apply, problems.py:28-33).
//
// kls_csr_spmv reproduces CsrMatrix.matvec (problems.py:127-136) bit for bit:
// numpy forms prod = data * x[indices] and np.add.reduceat over each row,
// which evaluates prod[s] + pairwise_sum(prod[s+1:e]) with numpy's pairwise
// summation (8-way unrolled blocks of <= 128, recursive halving above, a
// sequential loop from -0.0 below 8).  Every product and sum here is an
// explicitly rounded __dmul_rn / __dadd_rn so nvcc cannot contract them into
// FMAs.  Empty rows give +0.0 (np.zeros).
//
// kls_stencil7 reproduces StencilLaplace3D._matvec (problems.py:296-305): the
// x-slowest (nx, ny, nz) grid, y = 6 g minus the six Dirichlet neighbours in
// the reference's order (x-1, x+1, y-1, y+1, z-1, z+1).  For a row-sharded
// grid the neighbouring x-planes of other ranks come in through x_lo / x_hi.
#include "reduce.cuh"
#include "seg.cuh"
#include "stencil.cuh"
#include "stencil_tma.cuh"
#include "peer.cuh"

#include <cstdlib>

namespace {

using namespace kls;

__device__ __forceinline__ double csr_prod(const int32_t* __restrict__ col,
                                           const double* __restrict__ val,
                                           const double* __restrict__ x, int64_t i) {
  return __dmul_rn(__ldg(val + i), __ldg(x + __ldg(col + i)));
}

// numpy pairwise_sum of prod[s : s + n] (n >= 0)
__device__ double csr_pairwise(const int32_t* __restrict__ col, const double* __restrict__ val,
                               const double* __restrict__ x, int64_t s, int64_t n) {
  if (n < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, csr_prod(col, val, x, s + i));
    return r;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = csr_prod(col, val, x, s + k);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], csr_prod(col, val, x, s + i + k));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, csr_prod(col, val, x, s + i));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(csr_pairwise(col, val, x, s, n2), csr_pairwise(col, val, x, s + n2, n - n2));
}

// One warp per 32 consecutive rows.  The warp first copies the rows'
// contiguous slice of column indices and values into shared memory with
// coalesced loads (the 12 B/nnz stream is read once, in full sectors), then
// each lane forms its row's products — all gathers of a row issued together —
// and sums them in reduceat order: p0 + (((-0.0 + p1) + p2) + ...).  Rows
// longer than 8 entries, or warps whose slice exceeds the staging buffer,
// use the general pairwise routine on global memory.
constexpr int kSpmvStage = 32 * 8;  // staged entries per warp

__global__ void __launch_bounds__(kThreads) csr_spmv_kernel(const int64_t* __restrict__ rowptr,
                                                            const int32_t* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            int64_t nrows,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y) {
  __shared__ int32_t scol[kWarps][kSpmvStage];
  __shared__ double sval[kWarps][kSpmvStage];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * kWarps + warp) * 32; r0 < nrows;
       r0 += nwarps * 32) {
    const int64_t i = r0 + lane;
    const bool live = i < nrows;
    const int64_t s = live ? __ldg(rowptr + i) : 0;
    const int64_t e = live ? __ldg(rowptr + i + 1) : 0;
    const int64_t wlast = min(r0 + 32, nrows);
    const int64_t ws = __shfl_sync(0xffffffffu, s, 0);
    const int64_t we = __ldg(rowptr + wlast);
    const int64_t total = we - ws;
    const bool staged = total <= kSpmvStage;
    if (staged) {
      for (int64_t k = lane; k < total; k += 32) {
        scol[warp][k] = __ldg(col + ws + k);
        sval[warp][k] = __ldg(val + ws + k);
      }
    }
    __syncwarp();
    const int64_t n = e - s;
    double acc = 0.0;
    if (live && n > 0 && n <= 8) {
      int32_t c[8];
      double v[8];
      const int64_t o = s - ws;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (staged) {
          c[k] = k < n ? scol[warp][o + k] : 0;
          v[k] = k < n ? sval[warp][o + k] : 0.0;
        } else {
          c[k] = k < n ? __ldg(col + s + k) : 0;
          v[k] = k < n ? __ldg(val + s + k) : 0.0;
        }
      }
      double p[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k] = k < n ? __dmul_rn(v[k], __ldg(x + c[k])) : 0.0;
      double r = -0.0;
#pragma unroll
      for (int k = 1; k < 8; ++k)
        if (k < n) r = __dadd_rn(r, p[k]);
      acc = __dadd_rn(p[0], r);
    } else if (live && n > 8) {
      acc = __dadd_rn(csr_prod(col, val, x, s), csr_pairwise(col, val, x, s + 1, n - 1));
    }
    if (live) y[i] = acc;
    __syncwarp();
  }
}

// ELL copy of a CSR block for short-row operators (stencils, 5/7-point):
// entry k of row i at k * ld + i, so lane-consecutive rows read consecutive
// addresses (fully coalesced 4 B / 8 B streams).  Per-row entry order is the
// CSR order, so the product is still formed in reduceat order and stays
// bit-identical to CsrMatrix.matvec.
__global__ void csr_to_ell_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, int64_t nrows, int32_t width,
                                  int64_t ld, int32_t* __restrict__ ecol, double* __restrict__ eval,
                                  uint8_t* __restrict__ elen) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nrows;
       i += stride) {
    const int64_t s = rowptr[i];
    const int n = static_cast<int>(rowptr[i + 1] - s);
    elen[i] = static_cast<uint8_t>(n);
    for (int k = 0; k < width; ++k) {
      ecol[k * ld + i] = k < n ? col[s + k] : 0;
      eval[k * ld + i] = k < n ? val[s + k] : 0.0;
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kThreads) ell_spmv_kernel(const int32_t* __restrict__ ecol,
                                                            const double* __restrict__ eval,
                                                            const uint8_t* __restrict__ elen,
                                                            int64_t nrows, int64_t ld,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nrows;
       i += stride) {
    const int n = __ldg(elen + i);
    int32_t c[W];
    double v[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
      c[k] = k < n ? __ldg(ecol + k * ld + i) : 0;
      v[k] = k < n ? __ldg(eval + k * ld + i) : 0.0;
    }
    double p[W];
#pragma unroll
    for (int k = 0; k < W; ++k) p[k] = k < n ? __dmul_rn(v[k], __ldg(x + c[k])) : 0.0;
    double acc = 0.0;
    if (n > 0) {
      double r = -0.0;
#pragma unroll
      for (int k = 1; k < W; ++k)
        if (k < n) r = __dadd_rn(r, p[k]);
      acc = __dadd_rn(p[0], r);
    }
    y[i] = acc;
  }
}

// Software-pipelined ELL product (default): while a thread gathers x for
// row i it already has the ELL entries of its next row in flight, so the
// streaming loads (HBM) overlap the gathers (mostly L1/L2).  The entry
// streams bypass L1 (they are used once) to leave it to the x gathers.
// Same arithmetic, same order as ell_spmv_kernel: bit-identical.
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
__device__ __forceinline__ int ld_na_u8(const uint8_t* p) {
  uint16_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
  return static_cast<int>(v);
}

#ifndef KLS_ELL_BLOCKS
#define KLS_ELL_BLOCKS 4
#endif
constexpr int kEllBlocks = KLS_ELL_BLOCKS;

template <int W>
struct EllRow {
  int n;
  int32_t c[W];
  double v[W];
};

// The entry loads are predicated on the stored width (uniform, known up
// front), not on the row's length: padding slots hold (0, 0.0), and
// predicating on elen would make every row's loads wait for its elen byte
// (one more dependent memory latency per row: 5.9 -> 6.6 TB/s at m = 1.3e8).
// The row length still bounds the arithmetic (numpy's reduceat order).
// W is the stored width itself for widths 4..8 (no predicates, no spills),
// else the next instantiated size with slots >= width predicated off.
template <int W>
__device__ __forceinline__ void ell_fetch(EllRow<W>& r, const int32_t* ecol, const double* eval,
                                          const uint8_t* elen, int64_t ld, int64_t i, int width) {
  r.n = ld_na_u8(elen + i);
#pragma unroll
  for (int k = 0; k < W; ++k) {
    r.c[k] = k < width ? ld_na_s32(ecol + k * ld + i) : 0;
    r.v[k] = k < width ? ld_na_f64(eval + k * ld + i) : 0.0;
  }
}

// resident CTAs per SM of the pipelined kernel: two rows of W entries in
// registers must fit the 64K-register file without spilling
template <int W>
constexpr int ell_blocks() { return W >= 7 ? 3 : kEllBlocks; }

// x accessors of the pipelined ELL product: the rank's window as one array,
// or (peer) as three — column c of [lo halo | own rows | hi halo] lives at
// lo[c], own[c - nlo] or hi[c - nlo - nown], the halo parts being the
// neighbouring ranks' vectors read over NVLink.
struct XPlain {
  const double* x;
  __device__ __forceinline__ double operator()(int64_t c) const { return __ldg(x + c); }
};
struct XWindow {
  const double* lo;
  const double* own;
  const double* hi;
  int64_t nlo;
  int64_t nown;
  __device__ __forceinline__ double operator()(int64_t c) const {
    if (c < nlo) return __ldg(lo + c);
    c -= nlo;
    if (c < nown) return __ldg(own + c);
    return __ldg(hi + (c - nown));
  }
};

// Peer variant: a CTA first waits until the neighbours' "vector written"
// flags (this rank's halo flags) reach epoch.
struct PeerWait {
  const uint64_t* flag_lo;
  const uint64_t* flag_hi;
  uint64_t epoch;
  int* err;
};

template <int W, typename XA>
__global__ void __launch_bounds__(kThreads, ell_blocks<W>()) ell_spmv_pipe_kernel(
    const int32_t* __restrict__ ecol, const double* __restrict__ eval,
    const uint8_t* __restrict__ elen, int64_t nrows, int64_t ld, XA x,
    double* __restrict__ y, PeerWait pw, int width) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // the first row's entries (the operator's own arrays, never written by
  // the preceding kernels) are fetched before waiting for x: the loads
  // overlap the predecessor's tail under PDL
  EllRow<W> cur;
  cur.n = 0;
  if (i < nrows) ell_fetch<W>(cur, ecol, eval, elen, ld, i, width);
  pdl_wait();  // x from the preceding update (and y free to overwrite)
  if (pw.flag_lo != nullptr || pw.flag_hi != nullptr) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
      bool ok = true;
      if (pw.flag_lo != nullptr) ok = ok && peer::wait_flag(pw.flag_lo, pw.epoch);
      if (pw.flag_hi != nullptr) ok = ok && peer::wait_flag(pw.flag_hi, pw.epoch);
      s_ok = ok;
      if (!ok) *pw.err = 1;
    }
    __syncthreads();
    if (!s_ok) return;
  }
  if (i >= nrows) return;
  while (true) {
    const int64_t nx = i + stride;
    EllRow<W> nxt;
    nxt.n = 0;
    if (nx < nrows) ell_fetch<W>(nxt, ecol, eval, elen, ld, nx, width);
    double p[W];
#pragma unroll
    for (int k = 0; k < W; ++k) p[k] = k < cur.n ? __dmul_rn(cur.v[k], x(cur.c[k])) : 0.0;
    double acc = 0.0;
    if (cur.n > 0) {
      double r = -0.0;
#pragma unroll
      for (int k = 1; k < W; ++k)
        if (k < cur.n) r = __dadd_rn(r, p[k]);
      acc = __dadd_rn(p[0], r);
    }
    y[i] = acc;
    if (nx >= nrows) break;
    cur = nxt;
    i = nx;
  }
  pdl_trigger();
}

int grid_1d(int64_t n, int per_sm) {
  const int64_t blocks = ceil_div(n, kThreads);
  int g = static_cast<int>(std::min<int64_t>(blocks, (int64_t)per_sm * sm_count()));
  return g < 1 ? 1 : g;
}

template <int W, typename XA>
int launch_ell_w(const int32_t* ecol, const double* eval, const uint8_t* elen, int32_t width,
                 int64_t nrows, int64_t ld, XA x, double* y, PeerWait pw, cudaStream_t st) {
  // one wave of resident CTAs; each thread walks its rows with a one-row lookahead
  const int grid = grid_1d(nrows, ell_blocks<W>());
  return launch_dependent(ell_spmv_pipe_kernel<W, XA>, dim3(grid), dim3(kThreads), 0, st,
                          "ell_spmv_pipe_kernel", ecol, eval, elen, nrows, ld, x, y, pw, width);
}

template <typename XA>
int launch_ell_pipe(const int32_t* ecol, const double* eval, const uint8_t* elen, int32_t width,
                    int64_t nrows, int64_t ld, XA x, double* y, PeerWait pw, cudaStream_t st) {
  switch (width) {
    case 5: return launch_ell_w<5>(ecol, eval, elen, width, nrows, ld, x, y, pw, st);
    case 6: return launch_ell_w<6>(ecol, eval, elen, width, nrows, ld, x, y, pw, st);
    case 7: return launch_ell_w<7>(ecol, eval, elen, width, nrows, ld, x, y, pw, st);
    case 8: return launch_ell_w<8>(ecol, eval, elen, width, nrows, ld, x, y, pw, st);
    default: return launch_ell_w<4>(ecol, eval, elen, width, nrows, ld, x, y, pw, st);  // 1..4
  }
}

__global__ void __launch_bounds__(kTileZ * kTileY) stencil7_kernel(
    const double* __restrict__ x, const double* __restrict__ x_lo, const double* __restrict__ x_hi,
    double* __restrict__ y, int64_t nx, int32_t ny, int32_t nz, int32_t xchunk) {
  const int64_t xa = static_cast<int64_t>(blockIdx.z) * xchunk;
  const int64_t xb = xa + xchunk < nx ? xa + xchunk : nx;
  stencil7_march(x, x_lo, x_hi, y, nx, ny, nz, xa, xb);
}

__global__ void __launch_bounds__(32 * kSTY) stencil7_smem_kernel(
    const double* __restrict__ x, const double* __restrict__ x_lo, const double* __restrict__ x_hi,
    double* __restrict__ y, int64_t nx, int32_t ny, int32_t nz, int32_t xchunk) {
  __shared__ double tile[kSTY + 2][kSTZ + 2];
  pdl_wait();  // x from the preceding update
  const int64_t xa = static_cast<int64_t>(blockIdx.z) * xchunk;
  const int64_t xb = xa + xchunk < nx ? xa + xchunk : nx;
  if (xa >= xb) return;  // uniform per CTA: no thread reaches a barrier
  stencil7_tile_march(x, x_lo, x_hi, y, nx, ny, nz, xa, xb, tile);
  pdl_trigger();
}


// stencil variant: 2 = TMA-staged tiles (default), 1 = shared-memory tiles
// with register prefetch (KLS_STENCIL=smem), 0 = register march
// (KLS_STENCIL=reg); all bit-identical
int stencil_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("KLS_STENCIL");
    v = (e && e[0] == 'r') ? 0 : (e && e[0] == 's') ? 1 : 2;
  }
  return v;
}

// GMRES's per-column backward error (gmres.py:46-60, :171-172) on an ELL
// operator in one pass: y = A x row by row exactly as the pipelined product
// (same fetch, same arithmetic: y is bit-identical), never stored; the
// kernel accumulates ||b - y||^2, ||x||^2 and ||b||^2 and reduces them over
// the grid (deterministic).  Saves the write of y and the re-read of y, x
// and b by kls_resid_norms, and one launch per GMRES column.
// DUAL: the same pass also forms and stores y2 = A x2 (the step's operator
// product, bit-identical to kls_ell_spmv) from the entries already in
// registers -- the GMRES backward-error column riding on the step's apply.
template <int W, bool DUAL = false>
__global__ void __launch_bounds__(kThreads, W >= 7 ? 3 : 4) ell_resid_norms_kernel(
    const int32_t* __restrict__ ecol, const double* __restrict__ eval,
    const uint8_t* __restrict__ elen, int64_t ld, const double* __restrict__ x,
    const double* __restrict__ b, int width, const __grid_constant__ seg::SimpleArgs a,
    const double* __restrict__ x2, double* __restrict__ y2) {
  pdl_wait();
  seg::run_simple<kThreads, 3>(a, [&](int64_t r0, int64_t rows, int vi, int V, double (&v)[3]) {
    const int64_t stride = static_cast<int64_t>(V) * kThreads;
    int64_t i = r0 + static_cast<int64_t>(vi) * kThreads + threadIdx.x;
    const int64_t end = r0 + rows;
    if (i >= end) return;
    EllRow<W> cur;
    ell_fetch<W>(cur, ecol, eval, elen, ld, i, width);
    while (true) {
      const int64_t nx = i + stride;
      EllRow<W> nxt;
      nxt.n = 0;
      if (nx < end) ell_fetch<W>(nxt, ecol, eval, elen, ld, nx, width);
      double p[W];
#pragma unroll
      for (int k = 0; k < W; ++k) p[k] = k < cur.n ? __dmul_rn(cur.v[k], __ldg(x + cur.c[k])) : 0.0;
      double acc = 0.0;
      if (cur.n > 0) {
        double r = -0.0;
#pragma unroll
        for (int k = 1; k < W; ++k)
          if (k < cur.n) r = __dadd_rn(r, p[k]);
        acc = __dadd_rn(p[0], r);
      }
      if constexpr (DUAL) {
        double p2[W];
#pragma unroll
        for (int k = 0; k < W; ++k) p2[k] = k < cur.n ? __dmul_rn(cur.v[k], __ldg(x2 + cur.c[k])) : 0.0;
        double acc2 = 0.0;
        if (cur.n > 0) {
          double r2 = -0.0;
#pragma unroll
          for (int k = 1; k < W; ++k)
            if (k < cur.n) r2 = __dadd_rn(r2, p2[k]);
          acc2 = __dadd_rn(p2[0], r2);
        }
        y2[i] = acc2;
      }
      const double bi = __ldcs(b + i);
      const double xi = __ldg(x + i);
      const double rr = bi - acc;
      v[0] = fma(rr, rr, v[0]);
      v[1] = fma(xi, xi, v[1]);
      v[2] = fma(bi, bi, v[2]);
      if (nx >= end) break;
      cur = nxt;
      i = nx;
    }
  });
  pdl_trigger();
}

template <int W>
int launch_ell_resid(const int32_t* ecol, const double* eval, const uint8_t* elen, int32_t width,
                     int64_t ld, const double* x, const double* b, const seg::SimpleArgs& a,
                     cudaStream_t st, const double* x2 = nullptr, double* y2 = nullptr) {
  // one item per CTA up to 4 CTAs per SM (at m = 1e6 all 504 items resident)
  const int grid = std::max(1, std::min(a.P.nitems, 4 * sm_count()));
  if (x2 != nullptr)
    return launch_dependent(ell_resid_norms_kernel<W, true>, dim3(grid), dim3(kThreads), 0, st,
                            "ell_resid_norms_kernel", ecol, eval, elen, ld, x, b, width, a, x2, y2);
  return launch_dependent(ell_resid_norms_kernel<W>, dim3(grid), dim3(kThreads), 0, st,
                          "ell_resid_norms_kernel", ecol, eval, elen, ld, x, b, width, a,
                          static_cast<const double*>(nullptr), static_cast<double*>(nullptr));
}

// dense y = A x, A row-major n x n (DenseOperator, problems.py:68-85):
// one warp per row
__global__ void __launch_bounds__(kThreads) dense_gemv_kernel(const double* __restrict__ a,
                                                              int64_t lda, int64_t n,
                                                              const double* __restrict__ x,
                                                              double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n;
       r += warps) {
    double acc = 0.0;
    for (int64_t c = lane; c < n; c += 32) acc = fma(__ldg(a + r * lda + c), __ldg(x + c), acc);
    acc = warp_sum(acc);
    if (lane == 0) y[r] = acc;
  }
}


}  // namespace

// y(0:nrows) = A x for a CSR block (int64 row pointer, int32 column indices
// into x).  For a row-sharded operator the indices address the rank's
// extended vector [lo halo | local | hi halo].
KLS_API int kls_csr_spmv(const int64_t* rowptr, const int32_t* col, const double* val,
                         int64_t nrows, const double* x, double* y, void* stream) {
  if (nrows == 0) return KLS_OK;  // a rank without rows
  if (nrows < 0 || rowptr == nullptr || x == nullptr || y == nullptr)
    return fail(KLS_EINVAL, "csr_spmv: bad arguments");
  const int64_t blocks = ceil_div(nrows, 32 * kWarps);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(blocks, 8LL * sm_count())));
  csr_spmv_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(rowptr, col, val, nrows,
                                                                            x, y);
  return check_launch("csr_spmv_kernel");
}

// Matrix-free 7-point Laplacian on nx local x-planes of an (.., ny, nz) grid.
// x_lo / x_hi: the neighbouring planes owned by other ranks, or NULL at the
// physical (Dirichlet) boundary.
KLS_API int kls_stencil7(const double* x, const double* x_lo, const double* x_hi, double* y,
                         int64_t nx, int64_t ny, int64_t nz, void* stream) {
  if (nx * ny * nz == 0 && nx >= 0 && ny >= 0 && nz >= 0) return KLS_OK;
  if (x == nullptr || y == nullptr || nx < 0 || ny < 0 || nz < 0)
    return fail(KLS_EINVAL, "stencil7: bad arguments");
  const int64_t n = nx * ny * nz;
  if (ny > INT32_MAX || nz > INT32_MAX) return fail(KLS_EINVAL, "stencil7: ny, nz must fit int32");
  static int env_chunk = -1;
  if (env_chunk < 0) {
    const char* e = getenv("KLS_STENCIL_XCHUNK");
    env_chunk = e ? atoi(e) : 0;
  }
  dim3 grid;
  if (stencil_variant() == 2 && stencil7_tma_ok(x, ny, nz)) {
    const int64_t xc = std::min<int64_t>(env_chunk > 0 ? env_chunk : 32, nx);
    if (!stencil7_grid(nx, ny, nz, xc, grid, kTZ, kTY))
      return fail(KLS_EINVAL, "stencil7: grid too large");
    CUtensorMap map;
    const int use_map = stencil7_tensor_map(x, nx, ny, nz, &map) ? 1 : 0;
    TmaStencilArgs a{use_map, x, x_lo, x_hi, y, nx, static_cast<int32_t>(ny),
                     static_cast<int32_t>(nz), static_cast<int32_t>(xc), nullptr, nullptr, 0,
                     nullptr};
    return launch_dependent(stencil7_tma_kernel, grid, dim3(kTThreads), 0,
                            static_cast<cudaStream_t>(stream), "stencil7_tma_kernel", a, map);
  }
  if (stencil_variant() >= 1) {
    const int64_t xc = std::min<int64_t>(env_chunk > 0 ? env_chunk : 32, nx);
    if (!stencil7_grid(nx, ny, nz, xc, grid, kSTZ, kSTY))
      return fail(KLS_EINVAL, "stencil7: grid too large");
    return launch_dependent(stencil7_smem_kernel, grid, dim3(32, kSTY), 0,
                            static_cast<cudaStream_t>(stream), "stencil7_smem_kernel", x, x_lo,
                            x_hi, y, nx, static_cast<int32_t>(ny), static_cast<int32_t>(nz),
                            static_cast<int32_t>(xc));
  }
  const int64_t xchunk = std::min<int64_t>(env_chunk > 0 ? env_chunk : 16, nx);
  if (!stencil7_grid(nx, ny, nz, xchunk, grid)) return fail(KLS_EINVAL, "stencil7: grid too large");
  stencil7_kernel<<<grid, dim3(kTileZ, kTileY), 0, static_cast<cudaStream_t>(stream)>>>(
      x, x_lo, x_hi, y, nx, static_cast<int32_t>(ny), static_cast<int32_t>(nz),
      static_cast<int32_t>(xchunk));
  return check_launch("stencil7_kernel");
}

KLS_API int kls_dense_gemv(const double* a, int64_t lda, int64_t n, const double* x, double* y,
                           void* stream) {
  if (a == nullptr || x == nullptr || y == nullptr || n < 0 || lda < n)
    return fail(KLS_EINVAL, "dense_gemv: bad arguments");
  if (n == 0) return KLS_OK;
  const int64_t blocks = ceil_div(n, kWarps);
  const int grid = static_cast<int>(std::min<int64_t>(blocks, 8LL * sm_count()));
  dense_gemv_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, lda, n, x, y);
  return check_launch("dense_gemv_kernel");
}

// Convert a CSR block whose rows hold <= width (<= 8) entries to the ELL
// layout above (ecol / eval: width * ld entries, elen: nrows bytes).
KLS_API int kls_csr_to_ell(const int64_t* rowptr, const int32_t* col, const double* val,
                           int64_t nrows, int32_t width, int64_t ld, int32_t* ecol, double* eval,
                           uint8_t* elen, void* stream) {
  if (rowptr == nullptr || nrows < 0 || width < 1 || width > 8 || ld < nrows || ecol == nullptr ||
      eval == nullptr || elen == nullptr)
    return fail(KLS_EINVAL, "csr_to_ell: bad arguments");
  if (nrows == 0) return KLS_OK;
  csr_to_ell_kernel<<<grid_1d(nrows, 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      rowptr, col, val, nrows, width, ld, ecol, eval, elen);
  return check_launch("csr_to_ell_kernel");
}

// y = A x from the ELL layout; bit-identical to kls_csr_spmv on the same rows.
KLS_API int kls_ell_spmv(const int32_t* ecol, const double* eval, const uint8_t* elen,
                         int32_t width, int64_t nrows, int64_t ld, const double* x, double* y,
                         void* stream) {
  if (nrows == 0) return KLS_OK;
  if (ecol == nullptr || eval == nullptr || elen == nullptr || x == nullptr || y == nullptr ||
      nrows < 0 || ld < nrows || width < 1 || width > 8)
    return fail(KLS_EINVAL, "ell_spmv: bad arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static const bool plain = [] {
    const char* e = getenv("KLS_ELL");
    return e != nullptr && e[0] == 'p';
  }();
  if (plain) {
    const int grid = grid_1d(nrows, 8);
    if (width <= 4)
      ell_spmv_kernel<4><<<grid, kThreads, 0, st>>>(ecol, eval, elen, nrows, ld, x, y);
    else if (width <= 6)
      ell_spmv_kernel<6><<<grid, kThreads, 0, st>>>(ecol, eval, elen, nrows, ld, x, y);
    else
      ell_spmv_kernel<8><<<grid, kThreads, 0, st>>>(ecol, eval, elen, nrows, ld, x, y);
    return check_launch("ell_spmv_kernel");
  }
  return launch_ell_pipe(ecol, eval, elen, width, nrows, ld, XPlain{x}, y,
                         PeerWait{nullptr, nullptr, 0, nullptr}, st);
}

// out = [||b - A x||^2, ||x||^2, ||b||^2] over this row block for an ELL
// operator (rows of x at their own index: a one-rank operator), A x formed
// bit-identically to kls_ell_spmv but not stored.
KLS_API int kls_ell_resid_norms(const int32_t* ecol, const double* eval, const uint8_t* elen,
                                int32_t width, int64_t nrows, int64_t ld, const double* x,
                                const double* b, double* out, const KlsSegs* segs, void* ws,
                                size_t ws_bytes, void* stream) {
  if ((nrows > 0 && (ecol == nullptr || eval == nullptr || elen == nullptr || x == nullptr ||
                     b == nullptr)) ||
      out == nullptr || ws == nullptr || nrows < 0 || ld < nrows || width < 1 || width > 8)
    return fail(KLS_EINVAL, "ell_resid_norms: bad arguments");
  seg::SimpleArgs a;
  int rc = seg::make_plan_simple(segs, nrows, 2048, a, ws, ws_bytes, 3, out);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (width) {
    case 5: return launch_ell_resid<5>(ecol, eval, elen, width, ld, x, b, a, st);
    case 6: return launch_ell_resid<6>(ecol, eval, elen, width, ld, x, b, a, st);
    case 7: return launch_ell_resid<7>(ecol, eval, elen, width, ld, x, b, a, st);
    case 8: return launch_ell_resid<8>(ecol, eval, elen, width, ld, x, b, a, st);
    default: return launch_ell_resid<4>(ecol, eval, elen, width, ld, x, b, a, st);
  }
}

// The step's ELL product y2 = A x2 (bit-identical to kls_ell_spmv) and the
// backward-error norms of kls_ell_resid_norms for x (bit-identical too) in
// ONE pass over the operator's entries (GMRES, plan.cu).
KLS_API int kls_ell_apply_resid_norms(const int32_t* ecol, const double* eval,
                                      const uint8_t* elen, int32_t width, int64_t nrows,
                                      int64_t ld, const double* x2, double* y2, const double* x,
                                      const double* b, double* out, const KlsSegs* segs, void* ws,
                                      size_t ws_bytes, void* stream) {
  if ((nrows > 0 && (ecol == nullptr || eval == nullptr || elen == nullptr || x == nullptr ||
                     b == nullptr || x2 == nullptr || y2 == nullptr)) ||
      out == nullptr || ws == nullptr || nrows < 0 || ld < nrows || width < 1 || width > 8)
    return fail(KLS_EINVAL, "ell_apply_resid_norms: bad arguments");
  seg::SimpleArgs a;
  int rc = seg::make_plan_simple(segs, nrows, 2048, a, ws, ws_bytes, 3, out);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (width) {
    case 5: return launch_ell_resid<5>(ecol, eval, elen, width, ld, x, b, a, st, x2, y2);
    case 6: return launch_ell_resid<6>(ecol, eval, elen, width, ld, x, b, a, st, x2, y2);
    case 7: return launch_ell_resid<7>(ecol, eval, elen, width, ld, x, b, a, st, x2, y2);
    case 8: return launch_ell_resid<8>(ecol, eval, elen, width, ld, x, b, a, st, x2, y2);
    default: return launch_ell_resid<4>(ecol, eval, elen, width, ld, x, b, a, st, x2, y2);
  }
}

// kls_ell_spmv with the halo columns read from the neighbours' vectors over
// NVLink: x_lo = lower neighbour's rows [own_lo - nlo, own_lo) (peer-mapped),
// x_hi = upper neighbour's first rows (peer-mapped), either NULL when absent.
// Rows [b_lo, nrows - b_hi) touch only owned columns: they run first, with
// no wait and one plain gather per entry, overlapping the neighbours'
// progress; the b_lo leading and b_hi trailing rows then wait for this
// rank's halo flags from lo_rank / hi_rank (in mybuf) to reach epoch and
// read through the three-part window.  *err is set when a neighbour does not
// arrive within 20 s.  Same products and order: bit-identical to kls_ell_spmv.
KLS_API int kls_ell_spmv_peer(const int32_t* ecol, const double* eval, const uint8_t* elen,
                              int32_t width, int64_t nrows, int64_t ld, const double* x,
                              const double* x_lo, int64_t nlo, const double* x_hi, double* y,
                              int64_t b_lo, int64_t b_hi, void* mybuf, int32_t lo_rank,
                              int32_t hi_rank, uint64_t epoch, int* err, void* stream) {
  if (ecol == nullptr || eval == nullptr || elen == nullptr || x == nullptr || y == nullptr ||
      nrows < 0 || ld < nrows || width < 1 || width > 8 || mybuf == nullptr || err == nullptr ||
      (nlo > 0 && x_lo == nullptr) || nlo < 0 || lo_rank >= peer::kMaxPeers ||
      hi_rank >= peer::kMaxPeers || b_lo < 0 || b_hi < 0 || b_lo + b_hi > nrows)
    return fail(KLS_EINVAL, "ell_spmv_peer: bad arguments");
  if (nrows == 0) return KLS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(mybuf) + peer::kMaxPeers;
  const uint64_t* flo = (x_lo != nullptr && lo_rank >= 0) ? flags + lo_rank : nullptr;
  const uint64_t* fhi = (x_hi != nullptr && hi_rank >= 0) ? flags + hi_rank : nullptr;
  const PeerWait none{nullptr, nullptr, 0, nullptr};
  const int64_t mid = nrows - b_lo - b_hi;
  int rc = KLS_OK;
  if (mid > 0)  // window column c of an interior row is own row c - nlo
    rc = launch_ell_pipe(ecol + b_lo, eval + b_lo, elen + b_lo, width, mid, ld, XPlain{x - nlo},
                         y + b_lo, none, st);
  const XWindow xw{x_lo, x, x_hi, nlo, nrows};
  if (rc == KLS_OK && b_lo > 0)
    rc = launch_ell_pipe(ecol, eval, elen, width, b_lo, ld, xw, y, PeerWait{flo, fhi, epoch, err},
                         st);
  if (rc == KLS_OK && b_hi > 0) {
    const int64_t r0 = nrows - b_hi;
    rc = launch_ell_pipe(ecol + r0, eval + r0, elen + r0, width, b_hi, ld, xw, y + r0,
                         PeerWait{flo, fhi, epoch, err}, st);
  }
  return rc;
}
