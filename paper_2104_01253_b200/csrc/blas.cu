// Vector and tall-skinny kernels for the callers around the Arnoldi step:
// the normalisation q = u / alpha (arnoldi.py:391, :453; ortho.py:398),
// the GMRES residual and backward-error norms (gmres.py:46-60, :151), and
// the Krylov-Schur basis rotation V(:, a:b) <- V(:, a:b) Z (eig.py:237).
#include "reduce.cuh"

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

// out[0] = ||b - ax||^2, out[1] = ||x||^2, out[2] = ||b||^2 in one pass
__global__ void __launch_bounds__(kThreads) resid_norms_kernel(const double* __restrict__ b,
                                                               const double* __restrict__ ax,
                                                               const double* __restrict__ x,
                                                               int64_t n, RedWs ws,
                                                               double* out) {
  double v[3] = {0.0, 0.0, 0.0};
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const double bi = b[i];
    const double r = bi - ax[i];
    const double xi = x[i];
    v[0] = fma(r, r, v[0]);
    v[1] = fma(xi, xi, v[1]);
    v[2] = fma(bi, bi, v[2]);
  }
  grid_reduce_finish<3>(v, ws, out);
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

}  // namespace

KLS_API int kls_scale(const double* x, double* y, int64_t n, double alpha, int32_t mode,
                      void* stream) {
  if (x == nullptr || y == nullptr || n < 0) return fail(KLS_EINVAL, "scale: bad arguments");
  if (n == 0) return KLS_OK;
  scale_kernel<<<grid_1d(n, 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(x, y, n, alpha,
                                                                                mode);
  return check_launch("scale_kernel");
}

KLS_API int kls_sub(const double* a, const double* b, double* out, int64_t n, void* stream) {
  if (a == nullptr || b == nullptr || out == nullptr || n < 0)
    return fail(KLS_EINVAL, "sub: bad arguments");
  if (n == 0) return KLS_OK;
  sub_kernel<<<grid_1d(n, 8), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(a, b, out, n);
  return check_launch("sub_kernel");
}

KLS_API int kls_resid_norms(const double* b, const double* ax, const double* x, int64_t n,
                            double* out, void* ws, size_t ws_bytes, void* stream) {
  if (b == nullptr || ax == nullptr || x == nullptr || out == nullptr || ws == nullptr || n < 0)
    return fail(KLS_EINVAL, "resid_norms: bad arguments");
  const int grid = grid_1d(n, 4);
  if (!red_ws_fits(ws_bytes, grid, 3)) return fail(KLS_ENOSPC, "resid_norms: workspace too small");
  resid_norms_kernel<<<grid, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(b, ax, x, n,
                                                                               red_ws(ws), out);
  return check_launch("resid_norms_kernel");
}

KLS_API int kls_tsgemm_inplace(double* V, int64_t ldv, int64_t m, int32_t k, const double* Z,
                               void* stream) {
  if (V == nullptr || Z == nullptr || m < 0 || k < 0 || ldv < m)
    return fail(KLS_EINVAL, "tsgemm_inplace: bad arguments");
  if (m == 0 || k == 0) return KLS_OK;
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
