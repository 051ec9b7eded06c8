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
#include "stencil.cuh"

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

__global__ void __launch_bounds__(kThreads) csr_spmv_kernel(const int64_t* __restrict__ rowptr,
                                                            const int32_t* __restrict__ col,
                                                            const double* __restrict__ val,
                                                            int64_t nrows,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ y) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nrows;
       i += stride) {
    const int64_t s = __ldg(rowptr + i);
    const int64_t e = __ldg(rowptr + i + 1);
    double acc = 0.0;
    if (e > s) acc = __dadd_rn(csr_prod(col, val, x, s), csr_pairwise(col, val, x, s + 1, e - s - 1));
    y[i] = acc;
  }
}

__global__ void __launch_bounds__(kTileZ * kTileY) stencil7_kernel(
    const double* __restrict__ x, const double* __restrict__ x_lo, const double* __restrict__ x_hi,
    double* __restrict__ y, int64_t nx, int32_t ny, int32_t nz, int32_t xchunk) {
  const int64_t xa = static_cast<int64_t>(blockIdx.z) * xchunk;
  const int64_t xb = xa + xchunk < nx ? xa + xchunk : nx;
  stencil7_march(x, x_lo, x_hi, y, nx, ny, nz, xa, xb);
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

int grid_1d(int64_t n, int per_sm) {
  const int64_t blocks = ceil_div(n, kThreads);
  int g = static_cast<int>(std::min<int64_t>(blocks, (int64_t)per_sm * sm_count()));
  return g < 1 ? 1 : g;
}

}  // namespace

// y(0:nrows) = A x for a CSR block (int64 row pointer, int32 column indices
// into x).  For a row-sharded operator the indices address the rank's
// extended vector [lo halo | local | hi halo].
KLS_API int kls_csr_spmv(const int64_t* rowptr, const int32_t* col, const double* val,
                         int64_t nrows, const double* x, double* y, void* stream) {
  if (nrows < 0 || rowptr == nullptr || x == nullptr || y == nullptr)
    return fail(KLS_EINVAL, "csr_spmv: bad arguments");
  if (nrows == 0) return KLS_OK;
  csr_spmv_kernel<<<grid_1d(nrows, 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      rowptr, col, val, nrows, x, y);
  return check_launch("csr_spmv_kernel");
}

// Matrix-free 7-point Laplacian on nx local x-planes of an (.., ny, nz) grid.
// x_lo / x_hi: the neighbouring planes owned by other ranks, or NULL at the
// physical (Dirichlet) boundary.
KLS_API int kls_stencil7(const double* x, const double* x_lo, const double* x_hi, double* y,
                         int64_t nx, int64_t ny, int64_t nz, void* stream) {
  if (x == nullptr || y == nullptr || nx < 0 || ny < 0 || nz < 0)
    return fail(KLS_EINVAL, "stencil7: bad arguments");
  const int64_t n = nx * ny * nz;
  if (n == 0) return KLS_OK;
  if (ny > INT32_MAX || nz > INT32_MAX) return fail(KLS_EINVAL, "stencil7: ny, nz must fit int32");
  static int env_chunk = -1;
  if (env_chunk < 0) {
    const char* e = getenv("KLS_STENCIL_XCHUNK");
    env_chunk = e ? atoi(e) : 0;
  }
  const int64_t xchunk = std::min<int64_t>(env_chunk > 0 ? env_chunk : 16, nx);
  dim3 grid;
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
