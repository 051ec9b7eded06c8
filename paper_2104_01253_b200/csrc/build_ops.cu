// Device-side construction of the test operators' CSR (the
// reference assembles them on the host with COO + lexsort, problems.py:
// 98-117, 208-245, 307-331, which needs tens of GB of host memory at
// m = 1e7..1e8).  Each rank builds only its own row block, with column
// indices already relative to its extended-vector base.
//
// The result is entry-for-entry identical to the host path: same ascending
// column order per row, same values with the same rounding (Manteuffel
// off-diagonals diff*(-1) + conv*(+-1), diagonal diff*4; Laplacian 6 / -1),
// and int64 row pointers from closed-form prefix counts of each stencil
// direction (no scan pass).
#include "common.cuh"

namespace {

using namespace kls;

// entries in rows [0, g) of the 7-point Dirichlet Laplacian on (nx, ny, nz)
__device__ __forceinline__ int64_t lap7_before(int64_t g, int64_t nx, int64_t ny, int64_t nz) {
  const int64_t P = ny * nz;
  const int64_t X = g / P;
  const int64_t rem = g - X * P;
  const int64_t iy = rem / nz;
  const int64_t iz = rem - iy * nz;
  int64_t c = g;                                          // diagonals
  c += g - min(g, P);                                     // x-1: rows with X >= 1
  c += min(g, (nx - 1) * P);                              // x+1: rows with X < nx-1
  c += X * (ny - 1) * nz + max((int64_t)0, rem - nz);     // y-1
  c += X * (ny - 1) * nz + min(rem, (ny - 1) * nz);       // y+1
  c += X * ny * (nz - 1) + iy * (nz - 1) + max((int64_t)0, iz - 1);  // z-1
  c += X * ny * (nz - 1) + iy * (nz - 1) + min(iz, nz - 1);          // z+1
  return c;
}

__global__ void lap7_csr_kernel(int64_t row_lo, int64_t nrows, int64_t nx, int64_t ny,
                                int64_t nz, int64_t col_base, int64_t* __restrict__ rowptr,
                                int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t P = ny * nz;
  const int64_t base = lap7_before(row_lo, nx, ny, nz);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= nrows;
       r += stride) {
    const int64_t g = row_lo + r;
    int64_t e = lap7_before(g, nx, ny, nz) - base;
    rowptr[r] = e;
    if (r == nrows) continue;
    const int64_t X = g / P;
    const int64_t rem = g - X * P;
    const int64_t iy = rem / nz;
    const int64_t iz = rem - iy * nz;
    const int64_t cg = g - col_base;
    // ascending columns: g-P, g-nz, g-1, g, g+1, g+nz, g+P
    if (X > 0) { col[e] = static_cast<int32_t>(cg - P); val[e++] = -1.0; }
    if (iy > 0) { col[e] = static_cast<int32_t>(cg - nz); val[e++] = -1.0; }
    if (iz > 0) { col[e] = static_cast<int32_t>(cg - 1); val[e++] = -1.0; }
    col[e] = static_cast<int32_t>(cg);
    val[e++] = 6.0;
    if (iz + 1 < nz) { col[e] = static_cast<int32_t>(cg + 1); val[e++] = -1.0; }
    if (iy + 1 < ny) { col[e] = static_cast<int32_t>(cg + nz); val[e++] = -1.0; }
    if (X + 1 < nx) { col[e] = static_cast<int32_t>(cg + P); val[e] = -1.0; }
  }
}

// entries in rows [0, r) of the 5-point convection-diffusion operator, k x k
__device__ __forceinline__ int64_t mant5_before(int64_t r, int64_t k) {
  const int64_t blk = r / k;
  const int64_t i = r - blk * k;
  int64_t c = r;                                       // diagonals
  c += max((int64_t)0, r - k);                         // r-k: rows with blk >= 1
  c += blk * (k - 1) + max((int64_t)0, i - 1);         // r-1: rows with i >= 1
  c += blk * (k - 1) + min(i, k - 1);                  // r+1: rows with i < k-1
  c += min(r, (k - 1) * k);                            // r+k: rows with blk < k-1
  return c;
}

__global__ void mant5_csr_kernel(int64_t row_lo, int64_t nrows, int64_t k, int64_t col_base,
                                 double diff, double conv, int64_t* __restrict__ rowptr,
                                 int32_t* __restrict__ col, double* __restrict__ val) {
  const int64_t base = mant5_before(row_lo, k);
  const double lower = __dadd_rn(__dmul_rn(diff, -1.0), __dmul_rn(conv, -1.0));
  const double upper = __dadd_rn(__dmul_rn(diff, -1.0), __dmul_rn(conv, 1.0));
  const double diag = __dmul_rn(diff, 4.0);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= nrows;
       r += stride) {
    const int64_t g = row_lo + r;
    int64_t e = mant5_before(g, k) - base;
    rowptr[r] = e;
    if (r == nrows) continue;
    const int64_t blk = g / k;
    const int64_t i = g - blk * k;
    const int64_t cg = g - col_base;
    if (blk > 0) { col[e] = static_cast<int32_t>(cg - k); val[e++] = lower; }
    if (i > 0) { col[e] = static_cast<int32_t>(cg - 1); val[e++] = lower; }
    col[e] = static_cast<int32_t>(cg);
    val[e++] = diag;
    if (i + 1 < k) { col[e] = static_cast<int32_t>(cg + 1); val[e++] = upper; }
    if (blk + 1 < k) { col[e] = static_cast<int32_t>(cg + k); val[e] = upper; }
  }
}

// Banded random operator (config 5's Arnoldi variant): row
// i has exactly d entries, one in each of d equal slices of its window
// [max(0, i - b), min(m, i + b + 1)) -- distinct and already ascending --
// at a hashed column of the slice, with a hashed value in [-1, 1).  All
// integer arithmetic is mod 2^64 and the value is (h >> 11) * 2^-53 * 2 - 1
// (exact), so the host restatement (oracle.band_random_coo) produces the
// same entries bit for bit.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void band_csr_kernel(int64_t m, int64_t band, int32_t d, uint64_t seed,
                                int64_t row_lo, int64_t nrows, int64_t col_base,
                                int64_t* __restrict__ rowptr, int32_t* __restrict__ col,
                                double* __restrict__ val) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r <= nrows;
       r += stride) {
    rowptr[r] = r * d;
    if (r == nrows) continue;
    const int64_t i = row_lo + r;
    const int64_t lo = i - band > 0 ? i - band : 0;
    const int64_t hi = i + band + 1 < m ? i + band + 1 : m;
    const int64_t w = hi - lo;
    for (int k = 0; k < d; ++k) {
      const int64_t a = lo + w * k / d, b = lo + w * (k + 1) / d;
      const uint64_t h = mix64(seed * 0x9E3779B97F4A7C15ull + static_cast<uint64_t>(i) *
                               0xD1B54A32D192ED03ull + static_cast<uint64_t>(k));
      const int64_t c = a + static_cast<int64_t>((h >> 32) % static_cast<uint64_t>(b - a));
      const uint64_t h2 = mix64(h ^ 0x5DEECE66Dull);
      col[r * d + k] = static_cast<int32_t>(c - col_base);
      val[r * d + k] = static_cast<double>(h2 >> 11) * 0x1.0p-53 * 2.0 - 1.0;
    }
  }
}

int grid_rows(int64_t n) {
  const int64_t b = ceil_div(n + 1, kThreads);
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 16LL * sm_count())));
}

}  // namespace

// nnz of rows [row_lo, row_hi) of laplace3d(nx, ny, nz) in CSR form.
KLS_API int64_t kls_lap7_nnz(int64_t nx, int64_t ny, int64_t nz, int64_t row_lo, int64_t row_hi) {
  auto before = [&](int64_t g) {
    const int64_t P = ny * nz, X = g / P, rem = g - X * P, iy = rem / nz, iz = rem - iy * nz;
    int64_t c = g;
    c += g - std::min(g, P);
    c += std::min(g, (nx - 1) * P);
    c += X * (ny - 1) * nz + std::max<int64_t>(0, rem - nz);
    c += X * (ny - 1) * nz + std::min(rem, (ny - 1) * nz);
    c += X * ny * (nz - 1) + iy * (nz - 1) + std::max<int64_t>(0, iz - 1);
    c += X * ny * (nz - 1) + iy * (nz - 1) + std::min(iz, nz - 1);
    return c;
  };
  return before(row_hi) - before(row_lo);
}

// CSR of rows [row_lo, row_lo + nrows) of the 7-point Laplacian
// (StencilLaplace3D.to_csr, problems.py:307-331); columns relative to the
// global row col_base.  rowptr has nrows + 1 entries (starting at 0).
KLS_API int kls_build_lap7_csr(int64_t nx, int64_t ny, int64_t nz, int64_t row_lo, int64_t nrows,
                               int64_t col_base, int64_t* rowptr, int32_t* col, double* val,
                               void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || row_lo < 0 || nrows < 0 || row_lo + nrows > nx * ny * nz ||
      rowptr == nullptr || (nrows > 0 && (col == nullptr || val == nullptr)))
    return fail(KLS_EINVAL, "build_lap7_csr: bad arguments");
  lap7_csr_kernel<<<grid_rows(nrows), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      row_lo, nrows, nx, ny, nz, col_base, rowptr, col, val);
  return check_launch("lap7_csr_kernel");
}

// nnz of rows [row_lo, row_hi) of the k x k Manteuffel operator.
KLS_API int64_t kls_mant5_nnz(int64_t k, int64_t row_lo, int64_t row_hi) {
  auto before = [&](int64_t r) {
    const int64_t blk = r / k, i = r - blk * k;
    int64_t c = r;
    c += std::max<int64_t>(0, r - k);
    c += blk * (k - 1) + std::max<int64_t>(0, i - 1);
    c += blk * (k - 1) + std::min(i, k - 1);
    c += std::min(r, (k - 1) * k);
    return c;
  };
  return before(row_hi) - before(row_lo);
}

// CSR of rows [row_lo, row_lo + nrows) of (1/h^2) M + (beta/2h) N
// (manteuffel_build, problems.py:232-245) given diff = 1/h^2 and
// conv = beta/(2h) computed on the host exactly as the reference does.
KLS_API int kls_build_mant5_csr(int64_t k, int64_t row_lo, int64_t nrows, int64_t col_base,
                                double diff, double conv, int64_t* rowptr, int32_t* col,
                                double* val, void* stream) {
  if (k < 1 || row_lo < 0 || nrows < 0 || row_lo + nrows > k * k || rowptr == nullptr ||
      (nrows > 0 && (col == nullptr || val == nullptr)))
    return fail(KLS_EINVAL, "build_mant5_csr: bad arguments");
  mant5_csr_kernel<<<grid_rows(nrows), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      row_lo, nrows, k, col_base, diff, conv, rowptr, col, val);
  return check_launch("mant5_csr_kernel");
}

// CSR of rows [row_lo, row_lo + nrows) of the banded random operator of
// order m (half bandwidth band >= d - 1, d entries per row, seed); columns
// relative to the global row col_base; rowptr[r] = r * d.
KLS_API int kls_build_band_csr(int64_t m, int64_t band, int32_t d, uint64_t seed, int64_t row_lo,
                               int64_t nrows, int64_t col_base, int64_t* rowptr, int32_t* col,
                               double* val, void* stream) {
  if (m < 1 || d < 1 || band < 0 || 2 * band + 1 < d || (m < d) || row_lo < 0 || nrows < 0 ||
      row_lo + nrows > m || rowptr == nullptr || (nrows > 0 && (col == nullptr || val == nullptr)))
    return fail(KLS_EINVAL, "build_band_csr: bad arguments (need d <= min(m, 2 band + 1))");
  band_csr_kernel<<<grid_rows(nrows), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      m, band, d, seed, row_lo, nrows, col_base, rowptr, col, val);
  return check_launch("band_csr_kernel");
}
