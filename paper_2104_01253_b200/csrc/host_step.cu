// Host half of a DCGS2 Arnoldi step (arnoldi.py:367-420) in C++, with the
// reference's numpy arithmetic reproduced bit for bit: the two dot products
// and the Hessenberg-correction product go through the same OpenBLAS entry
// points numpy's dot / matmul call (the caller passes numpy's own
// cblas_ddot / cblas_dgemv, ILP64), with the same arguments; everything else
// is the same IEEE operations in the same order.  Host code only: it replaces
// ~10 us of per-step numpy / Python overhead at latency-bound sizes.
#include "common.cuh"

#include <cmath>

namespace {

typedef double (*ddot_fn)(int64_t n, const double* x, int64_t incx, const double* y,
                          int64_t incy);
typedef void (*dgemv_fn)(int order, int trans, int64_t m, int64_t n, double alpha,
                         const double* a, int64_t lda, const double* x, int64_t incx,
                         double beta, double* y, int64_t incy);

constexpr int kCblasColMajor = 102;
constexpr int kCblasTrans = 112;
constexpr double kEps = 2.220446049250313e-16;  // np.finfo(np.float64).eps

}  // namespace

// g = [c(0:j), beta, s(0:j), s_piv, aw.aw]; h is the expansion's C-order
// (capacity x capacity-1) Hessenberg buffer (row stride ldh).  Returns 0 for
// a regular step (t_full[0:j+1], k_next[0:j+1], res = [alpha, vscale]),
// 1 for a happy breakdown (column j-1 of H completed), 2 for the Pythagorean
// breakdown; -1 on bad arguments.
KLS_API int kls_dcgs2_host_step(const double* g, int32_t j, int64_t m, double wscale,
                                const double* k_prev, double* h, int64_t ldh, double* t_full,
                                double* k_next, double* res, void* ddot, void* dgemv) {
  if (g == nullptr || h == nullptr || t_full == nullptr || k_next == nullptr || res == nullptr ||
      ddot == nullptr || dgemv == nullptr || j < 0 || (j > 0 && k_prev == nullptr) || ldh < j)
    return -1;
  const ddot_fn dot = reinterpret_cast<ddot_fn>(ddot);
  const dgemv_fn gemv = reinterpret_cast<dgemv_fn>(dgemv);
  const double* c = g;
  const double beta = g[j];
  const double* s = g + j + 1;
  const double s_piv = g[2 * j + 1];
  const double aw_norm = std::sqrt(g[2 * j + 2]);
  const double bclip = (0.0 > beta) ? 0.0 : beta;  // Python max(beta, 0.0)
  if (!(std::sqrt(bclip) > kEps * std::sqrt(static_cast<double>(m)) * wscale)) {
    if (j > 0) {
      for (int i = 0; i < j; ++i) h[static_cast<int64_t>(i) * ldh + (j - 1)] = k_prev[i] + c[i];
      h[static_cast<int64_t>(j) * ldh + (j - 1)] = 0.0;
    }
    return 1;
  }
  // numpy's DOUBLE_dot: sum = 0.; sum += cblas_ddot(...)
  const double cc = 0.0 + (j > 0 ? dot(j, c, 1, c, 1) : 0.0);
  const double alpha_sq = beta - cc;
  if (!(alpha_sq > beta * kEps * kEps)) return 2;
  const double alpha = std::sqrt(alpha_sq);
  const double cs = 0.0 + (j > 0 ? dot(j, c, 1, s, 1) : 0.0);
  const double t_piv = (s_piv - cs) / (alpha * alpha);
  for (int i = 0; i < j; ++i) t_full[i] = s[i] / alpha;
  t_full[j] = t_piv;
  if (j > 0) {
    for (int i = 0; i < j; ++i) h[static_cast<int64_t>(i) * ldh + (j - 1)] = k_prev[i] + c[i];
    h[static_cast<int64_t>(j) * ldh + (j - 1)] = alpha;
  }
  // hc = h[:j+1, :j] @ c  (numpy matmul -> gemv: ColMajor, Trans, N=j, M=j+1)
  double hc_small[1] = {0.0};
  double* hc = k_next;  // computed in place: k_next = t_full - hc / alpha
  if (j > 0) {
    gemv(kCblasColMajor, kCblasTrans, j, j + 1, 1.0, h, ldh, c, 1, 0.0, hc, 1);
  } else {
    hc = hc_small;
  }
  for (int i = 0; i <= j; ++i) k_next[i] = t_full[i] - hc[i] / alpha;
  res[0] = alpha;
  res[1] = aw_norm / alpha;
  return 0;
}
