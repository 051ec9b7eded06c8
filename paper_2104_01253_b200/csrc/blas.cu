// Vector and tall-skinny kernels for the callers around the Arnoldi step:
// the normalisation q = u / alpha (arnoldi.py:391, :453; ortho.py:398),
// the GMRES residual and backward-error norms (gmres.py:46-60, :151), and
// the Krylov-Schur basis rotation V(:, a:b) <- V(:, a:b) Z (eig.py:237).
#include "reduce.cuh"
#include "seg.cuh"
#include "tma.cuh"

#include <cstdlib>

namespace {

using namespace kls;

int grid_1d(int64_t n, int per_sm) {
  const int64_t blocks = ceil_div(n, kThreads);
  int g = static_cast<int>(std::min<int64_t>(blocks, (int64_t)per_sm * sm_count()));
  return g < 1 ? 1 : g;
}

// y = x / alpha (mode 0, IEEE division as numpy's u / alpha) or x * alpha (1)
__global__ void scale_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n,
                             double alpha, int mode) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = mode == 0 ? x[i] / alpha : x[i] * alpha;
}

// out = a - b  (b - op.apply(x) in gmres.py:151 and backward_error)
__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b,
                           double* __restrict__ out, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = a[i] - b[i];
}

// out[0] = ||b - ax||^2, out[1] = ||x||^2, out[2] = ||b||^2 in one pass,
// reduced over the fixed segment tree (seg.cuh).  Thread t of virtual CTA v
// takes the segment's rows v * 256 + t, stepping by V * 256 -- the same
// grouping as the ELL-fused kernel (spmv.cu), so both give the same bits
// for the same A x.
__global__ void __launch_bounds__(kThreads) resid_norms_kernel(const double* __restrict__ b,
                                                               const double* __restrict__ ax,
                                                               const double* __restrict__ x,
                                                               const __grid_constant__ seg::SimpleArgs a) {
  seg::run_simple<kThreads, 3>(a, [&](int64_t r0, int64_t rows, int v, int V, double (&acc)[3]) {
    const int64_t step = static_cast<int64_t>(V) * kThreads;
    for (int64_t i = static_cast<int64_t>(v) * kThreads + threadIdx.x; i < rows; i += step) {
      const double bi = __ldcs(b + r0 + i);
      const double r = bi - __ldcs(ax + r0 + i);
      const double xi = __ldcs(x + r0 + i);
      acc[0] = fma(r, r, acc[0]);
      acc[1] = fma(xi, xi, acc[1]);
      acc[2] = fma(bi, bi, acc[2]);
    }
  });
}

// V(:, 0:k) <- V(:, 0:k) Z in place, Z k x k column-major (device).  A CTA
// stages a 32-row tile of all k columns in shared memory, so rows can be
// overwritten after the tile is read.
constexpr int kTileRows = 32;

__global__ void __launch_bounds__(kThreads) tsgemm_kernel(double* __restrict__ V, int64_t ldv,
                                                          int64_t m, int32_t k,
                                                          const double* __restrict__ Z,
                                                          int z_in_smem) {
  extern __shared__ double sm[];
  double* tile = sm;                       // [k][kTileRows]
  double* zs = sm + (size_t)k * kTileRows;  // [k][k] when z_in_smem
  if (z_in_smem)
    for (int i = threadIdx.x; i < k * k; i += kThreads) zs[i] = Z[i];
  const double* zz = z_in_smem ? zs : Z;
  const int64_t ntiles = (m + kTileRows - 1) / kTileRows;
  const int r = threadIdx.x % kTileRows;
  const int c0 = threadIdx.x / kTileRows;
  constexpr int kCstep = kThreads / kTileRows;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * kTileRows;
    __syncthreads();
    for (int c = c0; c < k; c += kCstep) {
      const int64_t row = row0 + r;
      tile[c * kTileRows + r] = row < m ? V[c * ldv + row] : 0.0;
    }
    __syncthreads();
    const int64_t row = row0 + r;
    for (int c = c0; c < k; c += kCstep) {
      double acc = 0.0;
      for (int i = 0; i < k; ++i) acc = fma(tile[i * kTileRows + r], zz[c * k + i], acc);
      if (row < m) V[c * ldv + row] = acc;
    }
  }
}

// V(:, 0:p) <- V(:, 0:k) Z(:, 0:p) in place, register-blocked.  A CTA
// stages a 128-row tile of all k columns (and Z, row-major with padded row
// length zp) in shared memory; lane l of warp w accumulates rows l + 32 r
// (r < 4) for the 4 adjacent columns 4w + 32 pass + (0..3), so each k-step
// costs 4 tile loads (conflict-free) and 2 double2 broadcast loads of Z for
// 16 FMAs — the naive one-output-per-thread form was shared-memory bound at
// 2 loads per FMA (~13x slower at m = 1e7, k = 60).
constexpr int kRotRows = 128;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(src_bytes)
               : "memory");
}

__global__ void __launch_bounds__(kThreads, 2)
    rotate_kernel(double* __restrict__ V, int64_t ldv, int64_t m, int32_t k, int32_t p,
                  const double* __restrict__ Z, int32_t zp, int32_t dbuf) {
  extern __shared__ __align__(16) double smr[];
  double* zs = smr;                                   // [k][zp]
  double* const tile0 = smr + static_cast<size_t>(k) * zp;  // [k][kRotRows], x2 when dbuf
  double* const tile1 = tile0 + static_cast<size_t>(k) * kRotRows;
  for (int i = threadIdx.x; i < k * zp; i += kThreads) {
    const int r = i / zp, c = i % zp;
    zs[i] = c < p ? Z[static_cast<int64_t>(c) * k + r] : 0.0;
  }
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t ntiles = (m + kRotRows - 1) / kRotRows;
  const int npass = (p + 31) / 32;
  // tile t's k columns into buf with 16-byte cp.async (rows past m zero-filled)
  auto load_tile = [&](int64_t t, double* buf) {
    const int64_t row0 = t * kRotRows;
    for (int i = threadIdx.x; i < k * (kRotRows / 2); i += kThreads) {
      const int c = i / (kRotRows / 2), r2 = 2 * (i % (kRotRows / 2));
      const int64_t row = row0 + r2;
      const double* col = V + static_cast<int64_t>(c) * ldv;
      const int bytes = row + 2 <= m ? 16 : (row < m ? 8 : 0);
      cp_async16(buf + c * kRotRows + r2, bytes ? col + row : col, bytes);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int it = 0;
  if (static_cast<int64_t>(blockIdx.x) < ntiles) load_tile(blockIdx.x, tile0);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int64_t row0 = t * kRotRows;
    const bool full = row0 + kRotRows <= m;
    double* tile = (dbuf && (it & 1)) ? tile1 : tile0;
    const int64_t tn = t + gridDim.x;
    if (dbuf && tn < ntiles) {
      // the next tile streams in while this one is multiplied (in place is
      // safe: the tiles are disjoint rows, each owned by one CTA)
      load_tile(tn, (it & 1) ? tile0 : tile1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // the tile (and Z) are staged
    for (int pass = 0; pass < npass; ++pass) {
      const int cb = pass * 32 + 4 * warp;
      if (cb >= p) continue;
      double acc[4][4];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
#pragma unroll 4
      for (int i = 0; i < k; ++i) {
        double tv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) tv[r] = tile[i * kRotRows + lane + 32 * r];
        const double2 z01 = *reinterpret_cast<const double2*>(zs + i * zp + cb);
        const double2 z23 = *reinterpret_cast<const double2*>(zs + i * zp + cb + 2);
        const double zv[4] = {z01.x, z01.y, z23.x, z23.y};
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = fma(tv[r], zv[c], acc[r][c]);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (cb + c >= p) break;
        double* dst = V + static_cast<int64_t>(cb + c) * ldv + row0;
#pragma unroll
        for (int r = 0; r < 4; ++r)
          if (full || row0 + lane + 32 * r < m) dst[lane + 32 * r] = acc[r][c];
      }
    }
    __syncthreads();  // this tile's readers are done before it is refilled
    if (!dbuf && tn < ntiles) load_tile(tn, tile0);
  }
}

// fp64 tensor-core (DMMA, mma.sync m8n8k4) form of the same rotation, for
// k <= 64: a producer warp streams 128-row tiles of all k columns into a
// 2-3 stage shared-memory ring with cp.async.bulk (mbarrier completion; its
// 32 lanes issue the k one-column copies together); each of the MW consumer
// warps (16 by default) owns 128 / MW rows of the tile and forms its
// (128 / MW) x 32 output block per pass as MT x 4 mma tiles, A fragments from the
// tile, B fragments from Z (shared, zero-padded to a multiple of 4 rows),
// accumulating in k order.  A lane (k-quad q = lane & 3, row r = lane >> 2)
// reads tile[(kk + q) * ld + r] and Z[(kk + q) * zp + r + 8 b]: with ld = 132
// and zp = 36 (mod 32 doubles: 4 and 4) the four k-quads land 8 banks
// apart, so the 64-bit fragment loads are conflict-free (ld = 136 / zp = 40
// gave 2-way conflicts: 115 M replays at config 4's shape, ncu -- removing
// them did not change the time: the kernel is bound elsewhere).
constexpr int kMmaRows = 128;
constexpr int kMmaLd = 132;
// MW consumer warps (+ the producer), each owning MT = 16 / MW * 1 m-tiles
// of 8 rows: 8 warps x 2 tiles or 16 warps x 1 tile per 128-row tile
template <int MW>
constexpr int mma_threads() { return (MW + 1) * 32; }

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int MW>
__global__ void __launch_bounds__(mma_threads<MW>(), 1)
    rotate_mma_kernel(double* __restrict__ V, int64_t ldv, int64_t m, int32_t k, int32_t p,
                      const double* __restrict__ Z, int32_t kp, int32_t zp, int32_t stages) {
  using namespace kls::tma;
  extern __shared__ __align__(128) unsigned char smr_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smr_raw);
  uint64_t* empty = full + 4;
  double* zs = reinterpret_cast<double*>(smr_raw + 128);         // [kp][zp]
  double* ring = zs + static_cast<size_t>(kp) * zp;              // [stages][kp][kMmaLd]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kp * zp; i += blockDim.x) {
    const int r = i / zp, c = i % zp;
    zs[i] = (r < k && c < p) ? Z[static_cast<int64_t>(c) * k + r] : 0.0;
  }
  // ring columns k..kp-1 are never loaded: zero (they meet zero rows of Z)
  for (int i = threadIdx.x; i < stages * (kp - k) * kMmaLd; i += blockDim.x) {
    const int st = i / ((kp - k) * kMmaLd), rem = i % ((kp - k) * kMmaLd);
    ring[(static_cast<size_t>(st) * kp + k) * kMmaLd + rem] = 0.0;
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) {
      mbar_init(full + st, 1);
      mbar_init(empty + st, MW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int64_t ntiles = (m + kMmaRows - 1) / kMmaRows;
  constexpr int MT = 16 / MW;  // m-tiles per warp
  if (warp == MW) {  // producer: a tile is k one-column copies of <= 1 KB,
    // issued by all 32 lanes (one thread issuing them was the bound: ~50 ns
    // per copy); lane 0 arms the stage's barrier before any copy lands
    uint32_t use = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++use) {
      const int st = use % stages;
      const uint32_t round = use / stages;
      const int64_t row0 = t * kMmaRows;
      const int64_t nr = m - row0 < kMmaRows ? m - row0 : kMmaRows;
      const uint32_t bytes = static_cast<uint32_t>(nr & ~int64_t(1)) * sizeof(double);
      if (lane == 0) {
        if (round >= 1) mbar_wait(empty + st, (round - 1) & 1);
        mbar_expect_tx(full + st, bytes * static_cast<uint32_t>(k));
      }
      __syncwarp();
      if (bytes)
        for (int c = lane; c < k; c += 32)
          bulk_g2s(ring + (static_cast<size_t>(st) * kp + c) * kMmaLd,
                   V + static_cast<int64_t>(c) * ldv + row0, bytes, full + st);
    }
    return;
  }
  const int npass = (p + 31) / 32;
  const int r_a = 8 * MT * warp + (lane >> 2);  // tile row of the A fragment (+8 per m-tile)
  const int kq = lane & 3;
  uint32_t use = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++use) {
    const int st = use % stages;
    mbar_wait(full + st, (use / stages) & 1);
    const double* tile = ring + static_cast<size_t>(st) * kp * kMmaLd;
    const int64_t row0 = t * kMmaRows;
    const int64_t nr = m - row0 < kMmaRows ? m - row0 : kMmaRows;
    if (nr & 1) {  // the odd last row is not in the bulk copy
      double* tw = ring + static_cast<size_t>(st) * kp * kMmaLd;
      for (int c = threadIdx.x; c < k; c += MW * 32)
        tw[c * kMmaLd + nr - 1] = V[static_cast<int64_t>(c) * ldv + row0 + nr - 1];
      asm volatile("bar.sync 1, %0;" ::"n"(MW * 32) : "memory");
    }
    for (int pass = 0; pass < npass; ++pass) {
      double acc[MT][4][2];
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      const double* zcol = zs + pass * 32 + (lane >> 2);
#pragma unroll 4
      for (int kk = 0; kk < kp; kk += 4) {
        const double* trow = tile + (kk + kq) * kMmaLd;
        double av[MT];
#pragma unroll
        for (int a = 0; a < MT; ++a) av[a] = trow[r_a + 8 * a];
        const double* zr = zcol + (kk + kq) * zp;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double bv = zr[8 * b];
#pragma unroll
          for (int a = 0; a < MT; ++a) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv);
        }
      }
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        const int64_t row = row0 + 8 * MT * warp + 8 * a + (lane >> 2);
        if (row >= m) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = pass * 32 + 8 * b + 2 * kq + e;
            if (col < p) V[static_cast<int64_t>(col) * ldv + row] = acc[a][b][e];
          }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
  }
}

// The same rotation on 256-row tiles whose columns arrive in stages of 32
// (kRot2Cols): a tile is two stages, each column copy 2 KB instead of 1 KB
// -- half the bulk copies per byte (their issue and processing set the pace
// of the 128-row kernel).  16 consumer warps own 16 rows each (two m-tiles);
// every output still accumulates its k terms in ascending order: the same
// bits as rotate_mma_kernel and the DFMA kernel.  ld = 260 (mod 32 = 4):
// conflict-free fragment loads as with 132.
constexpr int kRot2Rows = 256;
constexpr int kRot2Ld = 260;
constexpr int kRot2Cols = 32;
constexpr int kRot2Warps = 16;
constexpr int kRot2Threads = (kRot2Warps + 1) * 32;

__global__ void __launch_bounds__(kRot2Threads, 1)
    rotate_mma2_kernel(double* __restrict__ V, int64_t ldv, int64_t m, int32_t k, int32_t p,
                       const double* __restrict__ Z, int32_t kp, int32_t zp, int32_t stages) {
  using namespace kls::tma;
  extern __shared__ __align__(128) unsigned char smr_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smr_raw);
  uint64_t* empty = full + 4;
  double* zs = reinterpret_cast<double*>(smr_raw + 128);        // [kp][zp]
  double* ring = zs + static_cast<size_t>(kp) * zp;             // [stages][kRot2Cols][kRot2Ld]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (kp + kRot2Cols - 1) / kRot2Cols;  // column stages per tile
  for (int i = threadIdx.x; i < kp * zp; i += blockDim.x) {
    const int r = i / zp, c = i % zp;
    zs[i] = (r < k && c < p) ? Z[static_cast<int64_t>(c) * k + r] : 0.0;
  }
  // stage columns past k are never loaded: zero (they meet zero rows of Z)
  for (int i = threadIdx.x; i < stages * kRot2Cols * kRot2Ld; i += blockDim.x) ring[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) {
      mbar_init(full + st, 1);
      mbar_init(empty + st, kRot2Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int64_t ntiles = (m + kRot2Rows - 1) / kRot2Rows;
  if (warp == kRot2Warps) {  // producer: all 32 lanes issue a stage's column copies
    uint32_t use = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t row0 = t * kRot2Rows;
      const int64_t nr = m - row0 < kRot2Rows ? m - row0 : kRot2Rows;
      const uint32_t bytes = static_cast<uint32_t>(nr & ~int64_t(1)) * sizeof(double);
      for (int h = 0; h < nch; ++h, ++use) {
        const int st = use % stages;
        const uint32_t round = use / stages;
        const int c0 = h * kRot2Cols;
        const int nc = min(kRot2Cols, k - c0);
        if (lane == 0) {
          if (round >= 1) mbar_wait(empty + st, (round - 1) & 1);
          mbar_expect_tx(full + st, bytes * static_cast<uint32_t>(nc > 0 ? nc : 0));
        }
        __syncwarp();
        if (bytes)
          for (int c = lane; c < nc; c += 32)
            bulk_g2s(ring + (static_cast<size_t>(st) * kRot2Cols + c) * kRot2Ld,
                     V + static_cast<int64_t>(c0 + c) * ldv + row0, bytes, full + st);
      }
    }
    return;
  }
  const int npass = (p + 31) / 32;
  const int r_a = 16 * warp + (lane >> 2);  // tile row of the A fragment (+8 for the 2nd m-tile)
  const int kq = lane & 3;
  uint32_t use = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t row0 = t * kRot2Rows;
    const int64_t nr = m - row0 < kRot2Rows ? m - row0 : kRot2Rows;
    // npass > 1 (p > 32) would re-read the stages: this kernel takes p <= 32
    double acc[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int h = 0; h < nch; ++h, ++use) {
      const int st = use % stages;
      mbar_wait(full + st, (use / stages) & 1);
      const double* tile = ring + static_cast<size_t>(st) * kRot2Cols * kRot2Ld;
      const int c0 = h * kRot2Cols;
      if (nr & 1) {  // the odd last row is not in the bulk copy
        double* tw = ring + static_cast<size_t>(st) * kRot2Cols * kRot2Ld;
        for (int c = threadIdx.x; c < min(kRot2Cols, k - c0); c += kRot2Warps * 32)
          tw[c * kRot2Ld + nr - 1] = V[static_cast<int64_t>(c0 + c) * ldv + row0 + nr - 1];
        asm volatile("bar.sync 1, %0;" ::"n"(kRot2Warps * 32) : "memory");
      }
      const int kend = min(kRot2Cols, kp - c0);
      const double* zcol = zs + (lane >> 2);
#pragma unroll 4
      for (int kk = 0; kk < kend; kk += 4) {
        const double* trow = tile + (kk + kq) * kRot2Ld;
        const double a0 = trow[r_a], a1 = trow[r_a + 8];
        const double* zr = zcol + (c0 + kk + kq) * zp;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double bv = zr[8 * b];
          dmma884(acc[0][b][0], acc[0][b][1], a0, bv);
          dmma884(acc[1][b][0], acc[1][b][1], a1, bv);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + st);
    }
    (void)npass;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int64_t row = row0 + 16 * warp + 8 * a + (lane >> 2);
      if (row >= m) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * b + 2 * kq + e;
          if (col < p) V[static_cast<int64_t>(col) * ldv + row] = acc[a][b][e];
        }
    }
  }
}

size_t rotate_mma2_smem(int kp, int zp, int stages) {
  return 128 + sizeof(double) * (static_cast<size_t>(kp) * zp +
                                 static_cast<size_t>(stages) * kRot2Cols * kRot2Ld);
}

size_t rotate_mma_smem(int kp, int zp, int stages) {
  return 128 + sizeof(double) * (static_cast<size_t>(kp) * zp +
                                 static_cast<size_t>(stages) * kp * kMmaLd);
}

size_t rotate_smem(int k, int zp, int nbuf) {
  return sizeof(double) *
         (static_cast<size_t>(k) * zp + static_cast<size_t>(nbuf) * k * kRotRows);
}

}  // namespace

// V(:, 0:p) <- V(:, 0:k) Z(:, 0:p) in place (eig.py:237 keeps only the
// first p columns of V Z after the reordering); Z is k x p column-major
// (leading dimension k), on the device.  Columns p..k-1 of V are left as
// they were.
KLS_API int kls_tsgemm_inplace_cols(double* V, int64_t ldv, int64_t m, int32_t k, int32_t p,
                                    const double* Z, void* stream) {
  if (m == 0 && k >= 0 && p >= 0 && p <= k) return KLS_OK;  // a rank without rows
  if (V == nullptr || Z == nullptr || m < 0 || k < 0 || p < 0 || p > k || ldv < m)
    return fail(KLS_EINVAL, "tsgemm_inplace_cols: bad arguments");
  if (k == 0 || p == 0) return KLS_OK;
  static const bool use_mma = [] {  // KLS_ROTATE=fma: the DFMA kernel (experiments)
    const char* e = getenv("KLS_ROTATE");
    return !(e != nullptr && e[0] == 'f');
  }();
  {
    const int kp = (k + 3) / 4 * 4;
    const int zpm = (p + 31) / 32 * 32 + 4;  // B fragments conflict-free
    int stages = 3;
    while (stages > 1 && rotate_mma_smem(kp, zpm, stages) > 227 * 1024) --stages;
    // measured at m = 1e7 (scripts/rotate_probe.py): DMMA 1.35 vs DFMA 2.24 ms
    // at k = 60, p = 30; below k ~ 40 the DFMA kernel is faster (k = 30: 0.67
    // vs 0.89 ms).  Both accumulate each output in k order: identical bits.
    if (use_mma && k >= 40 && k <= 64 && stages >= 2 && (reinterpret_cast<uintptr_t>(V) & 15) == 0 &&
        (ldv & 1) == 0) {
      static const bool rot2 = [] {  // KLS_ROT2=0: the 128-row kernel (experiments)
        const char* e = getenv("KLS_ROT2");
        return !(e != nullptr && e[0] == '0');
      }();
      if (rot2 && p <= 32) {
        int st2 = 4;
        while (st2 > 2 && rotate_mma2_smem(kp, zpm, st2) > 220 * 1024) --st2;
        const size_t smem2 = rotate_mma2_smem(kp, zpm, st2);
        if (smem2 <= 220 * 1024) {
          cudaError_t e = cudaFuncSetAttribute(rotate_mma2_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem2));
          if (e != cudaSuccess) return fail(KLS_ECUDA, "rotate_mma2 smem: %s", cudaGetErrorString(e));
          const int grid2 = static_cast<int>(std::min<int64_t>(ceil_div(m, kRot2Rows), sm_count()));
          rotate_mma2_kernel<<<grid2, kRot2Threads, smem2, static_cast<cudaStream_t>(stream)>>>(
              V, ldv, m, k, p, Z, kp, zpm, st2);
          return check_launch("rotate_mma2_kernel");
        }
      }
      const size_t smem = rotate_mma_smem(kp, zpm, stages);
      // 16 consumer warps x 1 m-tile (4 per SM sub-partition to hide the
      // DMMA and fragment-load latency): 1.35 ms at config 4's shape, against
      // 1.45 with 8 warps x 2 tiles (KLS_ROT_WARPS=8, experiments)
      static const int mw = [] {
        const char* e = getenv("KLS_ROT_WARPS");
        return e != nullptr && atoi(e) == 8 ? 8 : 16;
      }();
      const void* fn = mw == 16 ? reinterpret_cast<const void*>(rotate_mma_kernel<16>)
                                : reinterpret_cast<const void*>(rotate_mma_kernel<8>);
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem));
      if (e != cudaSuccess) return fail(KLS_ECUDA, "rotate_mma smem: %s", cudaGetErrorString(e));
      const int grid = static_cast<int>(std::min<int64_t>(ceil_div(m, kMmaRows), sm_count()));
      if (mw == 16)
        rotate_mma_kernel<16><<<grid, mma_threads<16>(), smem, static_cast<cudaStream_t>(stream)>>>(
            V, ldv, m, k, p, Z, kp, zpm, stages);
      else
        rotate_mma_kernel<8><<<grid, mma_threads<8>(), smem, static_cast<cudaStream_t>(stream)>>>(
            V, ldv, m, k, p, Z, kp, zpm, stages);
      return check_launch("rotate_mma_kernel");
    }
  }
  const int zp = ((p + 31) / 32) * 32;
  const int dbuf = rotate_smem(k, zp, 2) <= 227 * 1024 ? 1 : 0;  // double-buffered tiles when they fit
  const size_t smem = rotate_smem(k, zp, dbuf ? 2 : 1);
  if ((reinterpret_cast<uintptr_t>(V) & 15) != 0 || (ldv & 1) != 0 || smem > 227 * 1024)
    return fail(KLS_EINVAL, "tsgemm_inplace_cols: V must be 16-byte aligned with even ldv, k <= %d",
                static_cast<int>((227 * 1024 / sizeof(double)) / (kRotRows + zp)));
  cudaError_t e = cudaFuncSetAttribute(rotate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return fail(KLS_ECUDA, "rotate smem: %s", cudaGetErrorString(e));
  const int64_t ntiles = ceil_div(m, kRotRows);
  const int per_sm = smem <= 110 * 1024 ? 2 : 1;
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, (int64_t)per_sm * sm_count()));
  rotate_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(V, ldv, m, k, p, Z,
                                                                            zp, dbuf);
  return check_launch("rotate_kernel");
}

KLS_API int kls_scale(const double* x, double* y, int64_t n, double alpha, int32_t mode,
                      void* stream) {
  if (n == 0) return KLS_OK;
  if (x == nullptr || y == nullptr || n < 0) return fail(KLS_EINVAL, "scale: bad arguments");
  scale_kernel<<<grid_1d(n, 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(x, y, n, alpha,
                                                                                mode);
  return check_launch("scale_kernel");
}

KLS_API int kls_sub(const double* a, const double* b, double* out, int64_t n, void* stream) {
  if (n == 0) return KLS_OK;
  if (a == nullptr || b == nullptr || out == nullptr || n < 0)
    return fail(KLS_EINVAL, "sub: bad arguments");
  sub_kernel<<<grid_1d(n, 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, b, out, n);
  return check_launch("sub_kernel");
}

KLS_API int kls_resid_norms(const double* b, const double* ax, const double* x, int64_t n,
                            double* out, const KlsSegs* segs, void* ws, size_t ws_bytes,
                            void* stream) {
  if ((n > 0 && (b == nullptr || ax == nullptr || x == nullptr)) || out == nullptr ||
      ws == nullptr || n < 0)
    return fail(KLS_EINVAL, "resid_norms: bad arguments");
  seg::SimpleArgs a;
  int rc = seg::make_plan_simple(segs, n, 2048, a, ws, ws_bytes, 3, out);
  if (rc) return rc;
  const int grid = std::max(1, std::min(a.P.nitems, 8 * sm_count()));
  resid_norms_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(b, ax, x, a);
  return check_launch("resid_norms_kernel");
}

KLS_API int kls_tsgemm_inplace(double* V, int64_t ldv, int64_t m, int32_t k, const double* Z,
                               void* stream) {
  if (V == nullptr || Z == nullptr || m < 0 || k < 0 || ldv < m)
    return fail(KLS_EINVAL, "tsgemm_inplace: bad arguments");
  if (m == 0 || k == 0) return KLS_OK;
  if ((reinterpret_cast<uintptr_t>(V) & 15) == 0 && (ldv & 1) == 0 &&
      rotate_smem(k, ((k + 31) / 32) * 32, 1) <= 227 * 1024)
    return kls_tsgemm_inplace_cols(V, ldv, m, k, k, Z, stream);
  size_t smem = sizeof(double) * (size_t)k * kTileRows;
  int z_in_smem = 0;
  if (smem + sizeof(double) * (size_t)k * k <= 200 * 1024) {
    smem += sizeof(double) * (size_t)k * k;
    z_in_smem = 1;
  }
  if (smem > 227 * 1024) return fail(KLS_EINVAL, "tsgemm_inplace: k=%d too large", k);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(tsgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return fail(KLS_ECUDA, "tsgemm smem: %s", cudaGetErrorString(e));
  }
  const int64_t ntiles = ceil_div(m, kTileRows);
  const int grid = static_cast<int>(std::min<int64_t>(ntiles, 2LL * sm_count()));
  tsgemm_kernel<<<grid, kThreads, smem, static_cast<cudaStream_t>(stream)>>>(V, ldv, m, k, Z,
                                                                            z_in_smem);
  return check_launch("tsgemm_kernel");
}
