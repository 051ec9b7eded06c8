// Microbenchmark: ELL (entry k of row i at k*ld + i: 2W separate streams)
// vs sliced ELL-32 (row block b, entry k, lane l at (b*W + k)*32 + l:
// one contiguous region per warp) for the 7-point operator's shape, with
// the x gather.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int W = 7;

__device__ __forceinline__ int64_t ell_idx(int64_t i, int k, int64_t ld) { return k * ld + i; }
__device__ __forceinline__ int64_t sell_idx(int64_t i, int k, int64_t) {
  return ((i >> 5) * W + k) * 32 + (i & 31);
}

template <bool SELL>
__global__ void __launch_bounds__(256, 4) spmv(const int* __restrict__ col, const double* __restrict__ val,
                                               const double* __restrict__ x, double* __restrict__ y,
                                               int64_t n, int64_t ld) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int c[W], cn[W];
  double v[W], vn[W];
  auto fetch = [&](int64_t r, int* cc, double* vv) {
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int64_t e = SELL ? sell_idx(r, k, ld) : ell_idx(r, k, ld);
      cc[k] = __ldcs(col + e);
      vv[k] = __ldcs(val + e);
    }
  };
  if (i < n) fetch(i, c, v);
  for (; i < n; i += stride) {
    const int64_t nx = i + stride;
    if (nx < n) fetch(nx, cn, vn);
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) acc += v[k] * __ldg(x + c[k]);
    y[i] = acc;
#pragma unroll
    for (int k = 0; k < W; ++k) c[k] = cn[k], v[k] = vn[k];
  }
}

__global__ void fill(int* col, double* val, int64_t n, int64_t ld, bool sell, int64_t nz, int64_t nyz) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t nb[W] = {i - nyz, i - nz, i - 1, i, i + 1, i + nz, i + nyz};
    for (int k = 0; k < W; ++k) {
      int64_t c = nb[k];
      if (c < 0 || c >= n) c = i;
      const int64_t e = sell ? ((i >> 5) * W + k) * 32 + (i & 31) : k * ld + i;
      col[e] = (int)c;
      val[e] = k == 3 ? 6.0 : -1.0;
    }
  }
}

int main() {
  const int64_t nx = 496, ny = 512, nz = 512, n = nx * ny * nz, ld = (n + 31) / 32 * 32;
  int* col;
  double *val, *x, *y;
  cudaMalloc(&col, sizeof(int) * W * ld);
  cudaMalloc(&val, sizeof(double) * W * ld);
  cudaMalloc(&x, sizeof(double) * n);
  cudaMalloc(&y, sizeof(double) * n);
  cudaMemset(x, 0, sizeof(double) * n);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)n * (W * 12 + 16);
  for (int rep = 0; rep < 2; ++rep)
    for (int sell = 0; sell < 2; ++sell) {
      fill<<<sms * 8, 256>>>(col, val, n, ld, sell, nz, ny * nz);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 3; ++w)
        sell ? spmv<true><<<sms * 4, 256>>>(col, val, x, y, n, ld) : spmv<false><<<sms * 4, 256>>>(col, val, x, y, n, ld);
      cudaEventRecord(a);
      for (int r = 0; r < 10; ++r)
        sell ? spmv<true><<<sms * 4, 256>>>(col, val, x, y, n, ld) : spmv<false><<<sms * 4, 256>>>(col, val, x, y, n, ld);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 10;
      printf("%s: %.3f ms  %.2f TB/s\n", sell ? "SELL-32" : "ELL    ", ms, bytes / ms / 1e9);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
