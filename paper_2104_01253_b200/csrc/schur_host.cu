// Host real-Schur services for Krylov-Schur restarts (reference schur.py) in
// C++, reproducing the reference's numpy arithmetic bit for bit so lock
// decisions are unchanged: every numpy operation that reaches BLAS / LAPACK
// (1-D dot, matmul as gemv / gemm, linalg.solve, linalg.qr) is issued to the
// same OpenBLAS entry points numpy uses (the caller passes numpy's own
// ILP64 scipy-openblas symbols) with the arguments numpy's dispatch chooses;
// everything else is the same IEEE operations in the same order.  Host code
// only: a restart's Francis sweeps run thousands of 3-row reflector
// applications, which cost ~2-4 ms here against ~100 ms as numpy calls.
//
// Matrices are C-order n x n (row stride n), as numpy's copies in schur.py.
#include "common.cuh"

#include <cmath>
#include <vector>

namespace {

typedef double (*ddot_fn)(int64_t n, const double* x, int64_t incx, const double* y,
                          int64_t incy);
typedef void (*dgemv_fn)(int order, int trans, int64_t m, int64_t n, double alpha,
                         const double* a, int64_t lda, const double* x, int64_t incx,
                         double beta, double* y, int64_t incy);
typedef void (*dgemm_fn)(int order, int ta, int tb, int64_t m, int64_t n, int64_t k,
                         double alpha, const double* a, int64_t lda, const double* b,
                         int64_t ldb, double beta, double* c, int64_t ldc);
typedef void (*dgesv_fn)(const int64_t* n, const int64_t* nrhs, double* a, const int64_t* lda,
                         int64_t* ipiv, double* b, const int64_t* ldb, int64_t* info);
typedef void (*dgeqrf_fn)(const int64_t* m, const int64_t* n, double* a, const int64_t* lda,
                          double* tau, double* work, const int64_t* lwork, int64_t* info);
typedef void (*zgemv_fn)(int order, int trans, int64_t m, int64_t n, const void* alpha,
                         const void* a, int64_t lda, const void* x, int64_t incx, const void* beta,
                         void* y, int64_t incy);
typedef void (*zdotu_fn)(int64_t n, const void* x, int64_t incx, const void* y, int64_t incy,
                         void* out);
typedef void (*dorgqr_fn)(const int64_t* m, const int64_t* n, const int64_t* k, double* a,
                          const int64_t* lda, const double* tau, double* work,
                          const int64_t* lwork, int64_t* info);

constexpr int kRowMajor = 101;
constexpr int kColMajor = 102;
constexpr int kNoTrans = 111;
constexpr int kTrans = 112;
constexpr double kEps = 2.220446049250313e-16;  // np.finfo(np.float64).eps

struct Blas {
  ddot_fn dot;
  dgemv_fn gemv;
  dgemm_fn gemm;
  dgesv_fn gesv;
  dgeqrf_fn geqrf;
  dorgqr_fn orgqr;
  zgemv_fn zgemv;
  zdotu_fn zdotu;
};

bool load(const KlsHostBlas* t, Blas* b) {
  if (t == nullptr || !t->ddot || !t->dgemv || !t->dgemm || !t->dgesv || !t->dgeqrf ||
      !t->dorgqr)
    return false;
  b->dot = reinterpret_cast<ddot_fn>(t->ddot);
  b->gemv = reinterpret_cast<dgemv_fn>(t->dgemv);
  b->gemm = reinterpret_cast<dgemm_fn>(t->dgemm);
  b->gesv = reinterpret_cast<dgesv_fn>(t->dgesv);
  b->geqrf = reinterpret_cast<dgeqrf_fn>(t->dgeqrf);
  b->orgqr = reinterpret_cast<dorgqr_fn>(t->dorgqr);
  b->zgemv = reinterpret_cast<zgemv_fn>(t->zgemv);
  b->zdotu = reinterpret_cast<zdotu_fn>(t->zdotu_sub);
  return true;
}

// ndarray.dot / np.dot of two 1-D float64 arrays (cblas_matrixproduct): a
// one-element operand is a "scalar" (a * b), otherwise DOUBLE_dot's
// sum = 0.; sum += cblas_ddot(...).
double npdot(const Blas& b, int64_t n, const double* x, int64_t incx, const double* y,
             int64_t incy) {
  if (n == 1) return y[0] * x[0];
  if (n <= 0) return 0.0;
  return 0.0 + b.dot(n, x, incx, y, incy);
}

// v @ A for A = rows x cols with row stride ld (a C-order block): numpy's
// vector_matrix special case -> cblas_dgemv(RowMajor, Trans, rows, cols, ..., lda = ld).
void vec_mat(const Blas& b, const double* v, const double* a, int64_t rows, int64_t cols,
             int64_t ld, double* out) {
  b.gemv(kRowMajor, kTrans, rows, cols, 1.0, a, ld, v, 1, 0.0, out, 1);
}

// A @ v, same block: matrix_vector -> cblas_dgemv(ColMajor, Trans, cols, rows, ..., lda = ld).
void mat_vec(const Blas& b, const double* a, int64_t rows, int64_t cols, int64_t ld,
             const double* v, double* out) {
  b.gemv(kColMajor, kTrans, cols, rows, 1.0, a, ld, v, 1, 0.0, out, 1);
}

// C-order block A (m x k, row stride lda) times B (k x p): matmul's
// matrix-matrix path -> cblas_dgemm(RowMajor, ...) into a fresh C-order
// m x p result.  ta: A is given as the transpose of a C-order k x m block.
void mat_mat(const Blas& b, bool ta, const double* a, int64_t lda, const double* bm,
             int64_t ldb, int64_t m, int64_t k, int64_t p, double* out) {
  b.gemm(kRowMajor, ta ? kTrans : kNoTrans, kNoTrans, m, p, k, 1.0, a, lda, bm, ldb, 0.0, out,
         p);
}

// numpy's pairwise summation (add.reduce over a contiguous run), from 0.
double pairwise_sum_abs(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += std::fabs(a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = std::fabs(a[k]);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += std::fabs(a[i + k]);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += std::fabs(a[i]);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sum_abs(a, n2) + pairwise_sum_abs(a + n2, n - n2);
}

// np.linalg.norm(T, ord=np.inf): row sums of |T|, then a NaN-propagating max
double norm_inf(const double* t, int64_t n) {
  double best = 0.0;
  for (int64_t r = 0; r < n; ++r) {
    const double s = 0.0 + pairwise_sum_abs(t + r * n, n);
    if (r == 0 || std::isnan(s) || (!std::isnan(best) && s > best)) best = s;
  }
  return best;
}

// Python max(a, b): a unless b > a.
inline double pymax(double a, double b) { return (b > a) ? b : a; }

// _reflector(x), x of length 2 or 3 (schur.py:139-155): v[0] = 1, beta.
void reflector(const Blas& b, const double* x, int len, double* v, double* beta) {
  double nrm = std::sqrt(npdot(b, len, x, 1, x, 1));
  if (nrm == 0.0) {
    for (int i = 0; i < len; ++i) v[i] = 0.0;
    *beta = 0.0;
    return;
  }
  if (x[0] > 0.0) nrm = -nrm;
  double u[3];
  for (int i = 0; i < len; ++i) u[i] = x[i];
  u[0] -= nrm;
  const double vv = npdot(b, len, u, 1, u, 1);
  if (vv == 0.0) {
    for (int i = 0; i < len; ++i) v[i] = 0.0;
    *beta = 0.0;
    return;
  }
  double bt = 2.0 / vv;
  const double lead = u[0];
  for (int i = 0; i < len; ++i) v[i] = u[i] / lead;
  bt *= lead * lead;
  *beta = bt;
}

// blk = T[r0:r0+len, c0:]; w = beta * (v @ blk); blk -= outer(v, w)
void reflect_rows(const Blas& b, double* t, int64_t n, const double* v, double beta, int64_t r0,
                  int64_t len, int64_t c0, std::vector<double>& w) {
  const int64_t cols = n - c0;
  double* blk = t + r0 * n + c0;
  vec_mat(b, v, blk, len, cols, n, w.data());
  for (int64_t c = 0; c < cols; ++c) w[c] = beta * w[c];
  for (int64_t i = 0; i < len; ++i)
    for (int64_t c = 0; c < cols; ++c) blk[i * n + c] -= v[i] * w[c];
}

// blk = M[:r1, c0:c0+len] (M n x n or Z); w = beta * (blk @ v); blk -= outer(w, v)
void reflect_cols(const Blas& b, double* t, int64_t n, const double* v, double beta, int64_t r1,
                  int64_t c0, int64_t len, std::vector<double>& w) {
  double* blk = t + c0;
  mat_vec(b, blk, r1, len, n, v, w.data());
  for (int64_t r = 0; r < r1; ++r) w[r] = beta * w[r];
  for (int64_t r = 0; r < r1; ++r)
    for (int64_t i = 0; i < len; ++i) blk[r * n + i] -= w[r] * v[i];
}

// split_block(T, Z, i) (schur.py:158-181)
void split_block(const Blas& b, double* t, double* z, int64_t n, int64_t i,
                 std::vector<double>& tmp) {
  const double a = t[i * n + i], bb = t[i * n + i + 1], c = t[(i + 1) * n + i],
               d = t[(i + 1) * n + i + 1];
  if (c == 0.0) return;
  const double half = 0.5 * (a - d);
  const double disc = half * half + bb * c;
  if (disc < 0.0) return;
  const double r = std::sqrt(disc);
  const double centre = 0.5 * (a + d);
  const double lam = half >= 0.0 ? centre + r : centre - r;
  const double ca[2] = {bb, lam - a};
  const double cb[2] = {lam - d, c};
  const double sa = std::fabs(ca[0]) + std::fabs(ca[1]);
  const double sb = std::fabs(cb[0]) + std::fabs(cb[1]);
  const double* v = sa >= sb ? ca : cb;
  const double nv = std::sqrt(npdot(b, 2, v, 1, v, 1));
  if (nv == 0.0) return;
  const double cs = v[0] / nv, sn = v[1] / nv;
  const double g[4] = {cs, -sn, sn, cs};  // C-order [[cs, -sn], [sn, cs]]
  const int64_t cols = n - i;
  if (static_cast<int64_t>(tmp.size()) < 2 * n) tmp.resize(2 * n);
  // T[i:i+2, i:] = G.T @ T[i:i+2, i:]
  mat_mat(b, true, g, 2, t + i * n + i, n, 2, 2, cols, tmp.data());
  for (int rr = 0; rr < 2; ++rr)
    for (int64_t cc = 0; cc < cols; ++cc) t[(i + rr) * n + i + cc] = tmp[rr * cols + cc];
  // T[:i+2, i:i+2] = T[:i+2, i:i+2] @ G
  mat_mat(b, false, t + i, n, g, 2, i + 2, 2, 2, tmp.data());
  for (int64_t rr = 0; rr < i + 2; ++rr)
    for (int cc = 0; cc < 2; ++cc) t[rr * n + i + cc] = tmp[rr * 2 + cc];
  // Z[:, i:i+2] = Z[:, i:i+2] @ G
  mat_mat(b, false, z + i, n, g, 2, n, 2, 2, tmp.data());
  for (int64_t rr = 0; rr < n; ++rr)
    for (int cc = 0; cc < 2; ++cc) z[rr * n + i + cc] = tmp[rr * 2 + cc];
  t[(i + 1) * n + i] = 0.0;
}

// _shifts (schur.py:184-203)
void shifts(const double* t, int64_t n, int64_t hi, int64_t stall, double* out) {
  auto T = [&](int64_t r, int64_t c) { return t[r * n + c]; };
  if (stall % 10 == 0) {
    const double w = std::fabs(T(hi, hi - 1)) + std::fabs(T(hi - 1, hi - 2));
    const double re = 0.75 * w + T(hi, hi);
    out[0] = re, out[1] = 0.0, out[2] = re, out[3] = 0.0;
    return;
  }
  const double a = T(hi - 1, hi - 1), b = T(hi - 1, hi), c = T(hi, hi - 1), d = T(hi, hi);
  const double sc = std::fabs(a) + std::fabs(b) + std::fabs(c) + std::fabs(d);
  if (sc == 0.0) {
    out[0] = out[1] = out[2] = out[3] = 0.0;
    return;
  }
  const double half = 0.5 * (a / sc - d / sc);
  const double disc = half * half + (b / sc) * (c / sc);
  const double centre = 0.5 * (a / sc + d / sc);
  if (disc >= 0.0) {
    const double r = std::sqrt(disc);
    const double r1 = centre + r, r2 = centre - r;
    const double pick = std::fabs(r1 - d / sc) <= std::fabs(r2 - d / sc) ? r1 : r2;
    out[0] = pick * sc, out[1] = 0.0, out[2] = pick * sc, out[3] = 0.0;
    return;
  }
  const double im = std::sqrt(-disc) * sc;
  out[0] = centre * sc, out[1] = im, out[2] = centre * sc, out[3] = -im;
}

// _francis_sweeps (schur.py:206-269); returns false on the sweep limit.
bool francis_sweeps(const Blas& b, double* t, double* z, int64_t n, int64_t max_sweeps) {
  std::vector<double> w(n + 4);
  auto T = [&](int64_t r, int64_t c) -> double& { return t[r * n + c]; };
  int64_t hi = n - 1;
  int64_t sweeps = 0, stall = 0;
  while (hi > 0) {
    int64_t lo = hi;
    while (lo > 0) {
      double s = std::fabs(T(lo - 1, lo - 1)) + std::fabs(T(lo, lo));
      if (s == 0.0) s = norm_inf(t, n);
      if (std::fabs(T(lo, lo - 1)) <= kEps * s) {
        T(lo, lo - 1) = 0.0;
        break;
      }
      lo -= 1;
    }
    if (lo == hi) {
      hi -= 1;
      stall = 0;
      continue;
    }
    if (lo == hi - 1) {
      split_block(b, t, z, n, lo, w);
      hi -= 2;
      stall = 0;
      continue;
    }
    sweeps += 1;
    stall += 1;
    if (sweeps > max_sweeps) return false;
    double sh[4];
    shifts(t, n, hi, stall, sh);
    const double re1 = sh[0], im1 = sh[1], re2 = sh[2], im2 = sh[3];
    const double h11 = T(lo, lo), h12 = T(lo, lo + 1), h21 = T(lo + 1, lo),
                 h22 = T(lo + 1, lo + 1);
    double sc = std::fabs(h11 - re2) + std::fabs(im2) + std::fabs(h21);
    if (sc == 0.0) sc = 1.0;
    const double h21s = h21 / sc;
    double col[3] = {h21s * h12 + (h11 - re1) * ((h11 - re2) / sc) - im1 * (im2 / sc),
                     h21s * (h11 + h22 - re1 - re2), h21s * T(lo + 2, lo + 1)};
    int clen = 3;
    double v[3], beta;
    for (int64_t k = lo; k < hi - 1; ++k) {
      reflector(b, col, clen, v, &beta);
      if (beta != 0.0) {
        reflect_rows(b, t, n, v, beta, k, 3, std::max(lo, k - 1), w);
        reflect_cols(b, t, n, v, beta, std::min(hi, k + 3) + 1, k, 3, w);
        reflect_cols(b, z, n, v, beta, n, k, 3, w);
      }
      if (k > lo) {
        T(k + 1, k - 1) = 0.0;
        T(std::min(k + 2, hi), k - 1) = 0.0;
      }
      clen = static_cast<int>(std::min<int64_t>(3, n - (k + 1)));
      for (int i = 0; i < clen; ++i) col[i] = T(k + 1 + i, k);
      if (k + 3 > hi) clen = std::min(clen, 2);
    }
    reflector(b, col, clen, v, &beta);
    if (beta != 0.0) {
      const int64_t k = hi - 1;
      reflect_rows(b, t, n, v, beta, k, 2, k - 1, w);
      reflect_cols(b, t, n, v, beta, hi + 1, k, 2, w);
      reflect_cols(b, z, n, v, beta, n, k, 2, w);
      T(hi, hi - 2) = 0.0;
    }
  }
  return true;
}

void block_list(const double* t, int64_t n, std::vector<int64_t>& b0, std::vector<int>& sz) {
  b0.clear();
  sz.clear();
  int64_t i = 0;
  while (i < n) {
    const int s = (i + 1 < n && t[(i + 1) * n + i] != 0.0) ? 2 : 1;
    b0.push_back(i);
    sz.push_back(s);
    i += s;
  }
}

double frob(const Blas& b, const double* a, int64_t rows, int64_t cols, int64_t ld) {
  // np.linalg.norm(block): ravel(order="K") (a C-order copy) then x.dot(x)
  double buf[16];
  int64_t k = 0;
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < cols; ++c) buf[k++] = a[r * ld + c];
  return std::sqrt(npdot(b, k, buf, 1, buf, 1));
}

// swap_adjacent_blocks (schur.py:294-319): 1 swapped, 0 refused.
int swap_blocks(const Blas& b, double* t, double* z, int64_t n, int64_t i, int p, int q,
                std::vector<double>& tmp) {
  const int s = p + q;
  double t11[4], t12[4], t22[4];
  for (int r = 0; r < p; ++r)
    for (int c = 0; c < p; ++c) t11[r * p + c] = t[(i + r) * n + i + c];
  for (int r = 0; r < p; ++r)
    for (int c = 0; c < q; ++c) t12[r * q + c] = t[(i + r) * n + i + p + c];
  for (int r = 0; r < q; ++r)
    for (int c = 0; c < q; ++c) t22[r * q + c] = t[(i + p + r) * n + i + p + c];
  // kron = kron(eye(q), t11) - kron(t22.T, eye(p)), (pq x pq), C-order
  const int pq = p * q;
  double kr[16];
  for (int ii = 0; ii < q; ++ii)
    for (int kk = 0; kk < p; ++kk)
      for (int jj = 0; jj < q; ++jj)
        for (int ll = 0; ll < p; ++ll) {
          const double e1 = (ii == jj) ? 1.0 : 0.0;
          const double e2 = (kk == ll) ? 1.0 : 0.0;
          const double k1 = e1 * t11[kk * p + ll];
          const double k2 = t22[jj * q + ii] * e2;  // t22.T[ii, jj]
          kr[(ii * p + kk) * pq + (jj * p + ll)] = k1 - k2;
        }
  // np.linalg.solve(kron, t12.reshape(-1, order="F")) -> dgesv on a Fortran copy
  double af[16], x[4];
  for (int r = 0; r < pq; ++r)
    for (int c = 0; c < pq; ++c) af[c * pq + r] = kr[r * pq + c];
  for (int c = 0; c < q; ++c)
    for (int r = 0; r < p; ++r) x[c * p + r] = t12[r * q + c];
  {
    int64_t nn = pq, nrhs = 1, lda = pq, ldb = pq, info = 0;
    int64_t ipiv[4];
    b.gesv(&nn, &nrhs, af, &lda, ipiv, x, &ldb, &info);
    if (info > 0) return 0;  // LinAlgError("Singular matrix")
    if (info < 0) return -1;
  }
  // X = x.reshape((p, q), order="F"); M = vstack([-X, eye(q)]) ((p+q) x q)
  // np.linalg.qr(M, mode="complete"): dgeqrf on a Fortran copy, then dorgqr
  // into a (p+q) x (p+q) Q (s > q always).
  double qf[16], tau[2];
  for (int c = 0; c < q; ++c) {
    for (int r = 0; r < p; ++r) qf[c * s + r] = -x[c * p + r];
    for (int r = 0; r < q; ++r) qf[c * s + p + r] = (r == c) ? 1.0 : 0.0;
  }
  {
    int64_t mm = s, nn = q, lda = s, lwork = -1, info = 0;
    double wq = 0.0;
    b.geqrf(&mm, &nn, qf, &lda, tau, &wq, &lwork, &info);
    int64_t lw = static_cast<int64_t>(wq);
    if (lw < nn) lw = nn;
    if (lw < 1) lw = 1;
    std::vector<double> work(lw);
    b.geqrf(&mm, &nn, qf, &lda, tau, work.data(), &lw, &info);
    if (info != 0) return -1;
    int64_t mc = s, kk = q;
    lwork = -1;
    b.orgqr(&mm, &mc, &kk, qf, &lda, tau, &wq, &lwork, &info);
    lw = static_cast<int64_t>(wq);
    if (lw < mc) lw = mc;
    if (lw < 1) lw = 1;
    work.assign(lw, 0.0);
    b.orgqr(&mm, &mc, &kk, qf, &lda, tau, work.data(), &lw, &info);
    if (info != 0) return -1;
  }
  // Qf as numpy holds it: C-order s x s
  double Q[16];
  for (int r = 0; r < s; ++r)
    for (int c = 0; c < s; ++c) Q[r * s + c] = qf[c * s + r];
  // rotated = Qf.T @ T[win, win] @ Qf
  double tmp1[16], rot[16];
  mat_mat(b, true, Q, s, t + i * n + i, n, s, s, s, tmp1);
  mat_mat(b, false, tmp1, s, Q, s, s, s, s, rot);
  const double lhs = frob(b, rot + q * s, p, q, s);
  const double tn = frob(b, t + i * n + i, s, s, n);
  if (lhs > 1e-8 * pymax(tn, 1.0)) return 0;
  const int64_t cols = n - i;
  if (static_cast<int64_t>(tmp.size()) < s * n) tmp.resize(s * n);
  // T[win, i:] = Qf.T @ T[win, i:]
  mat_mat(b, true, Q, s, t + i * n + i, n, s, s, cols, tmp.data());
  for (int r = 0; r < s; ++r)
    for (int64_t c = 0; c < cols; ++c) t[(i + r) * n + i + c] = tmp[r * cols + c];
  // T[:i+s, win] = T[:i+s, win] @ Qf
  mat_mat(b, false, t + i, n, Q, s, i + s, s, s, tmp.data());
  for (int64_t r = 0; r < i + s; ++r)
    for (int c = 0; c < s; ++c) t[r * n + i + c] = tmp[r * s + c];
  // Z[:, win] = Z[:, win] @ Qf
  mat_mat(b, false, z + i, n, Q, s, n, s, s, tmp.data());
  for (int64_t r = 0; r < n; ++r)
    for (int c = 0; c < s; ++c) z[r * n + i + c] = tmp[r * s + c];
  for (int r = i + q; r < i + s; ++r)
    for (int64_t c = i; c < i + q; ++c) t[r * n + c] = 0.0;
  if (q == 2) split_block(b, t, z, n, i, tmp);
  if (p == 2) split_block(b, t, z, n, i + q, tmp);
  return 1;
}

// ---- complex helpers: numpy complex128 arithmetic (loops.c.src) ----
struct Cx {
  double re, im;
};
inline Cx cx(double r, double i = 0.0) { return Cx{r, i}; }
inline Cx csub(Cx a, Cx b) { return Cx{a.re - b.re, a.im - b.im}; }
inline Cx cmul(Cx a, Cx b) { return Cx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
inline Cx cdiv(Cx a, Cx b) {  // CDOUBLE_divide (Smith)
  const double br = std::fabs(b.re), bi = std::fabs(b.im);
  if (br >= bi) {
    if (br == 0 && bi == 0) return Cx{a.re / br, a.im / br};
    const double rat = b.im / b.re;
    const double scl = 1.0 / (b.re + b.im * rat);
    return Cx{(a.re + a.im * rat) * scl, (a.im - a.re * rat) * scl};
  }
  const double rat = b.re / b.im;
  const double scl = 1.0 / (b.im + b.re * rat);
  return Cx{(a.re * rat + a.im) * scl, (a.im * rat - a.re) * scl};
}
inline double cabs_(Cx a) { return std::hypot(a.re, a.im); }  // npy_cabs

// real block A (rows x k, row stride ld) @ complex x (k): numpy casts A to a
// C-order complex copy, then matmul picks dot / noblas / zgemv by shape.
void rmat_cvec(const Blas& b, const double* a, int64_t rows, int64_t k, int64_t ld, const Cx* x,
               Cx* out, std::vector<Cx>& buf) {
  if (rows == 0) return;
  if (k == 0) {  // any_zero_dim: noblas -> zeros
    for (int64_t r = 0; r < rows; ++r) out[r] = cx(0.0);
    return;
  }
  if (static_cast<int64_t>(buf.size()) < rows * k) buf.resize(rows * k);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t c = 0; c < k; ++c) buf[r * k + c] = cx(a[r * ld + c]);
  if (rows == 1) {  // scalar_out: CDOUBLE_dot -> cblas_zdotu_sub, sum from 0
    double t[2];
    b.zdotu(k, buf.data(), 1, x, 1, t);
    out[0] = Cx{0.0 + t[0], 0.0 + t[1]};
    return;
  }
  if (k == 1) {  // scalar_vec: the noblas loop
    for (int64_t r = 0; r < rows; ++r) {
      const Cx v1 = buf[r], v2 = x[0];
      double re = 0.0, im = 0.0;
      re += (v1.re * v2.re) - (v1.im * v2.im);
      im += (v1.re * v2.im) + (v1.im * v2.re);
      out[r] = Cx{re, im};
    }
    return;
  }
  const double one[2] = {1.0, 0.0}, zero[2] = {0.0, 0.0};  // matrix_vector -> zgemv
  b.zgemv(kColMajor, kTrans, k, rows, one, buf.data(), k, x, 1, zero, out, 1);
}

// _back_substitute(T[:n0, :n0], lam, rhs) (schur.py:413-443); t has row stride ld.
void back_substitute(const Blas& b, const double* t, int64_t n0, int64_t ld, Cx lam,
                     const Cx* rhs, Cx* x, std::vector<Cx>& buf) {
  for (int64_t i = 0; i < n0; ++i) x[i] = cx(0.0);
  if (n0 == 0) return;
  // np.linalg.norm(T, ord=np.inf) of the (strided) block
  double nrm = 0.0;
  {
    std::vector<double> row(n0);
    for (int64_t r = 0; r < n0; ++r) {
      for (int64_t c = 0; c < n0; ++c) row[c] = t[r * ld + c];
      const double sr = 0.0 + pairwise_sum_abs(row.data(), n0);
      if (r == 0 || std::isnan(sr) || (!std::isnan(nrm) && sr > nrm)) nrm = sr;
    }
  }
  double big = nrm;  // Python max(nrm, abs(lam), 1.0)
  const double al = cabs_(lam);
  if (al > big) big = al;
  if (1.0 > big) big = 1.0;
  const double tiny = kEps * big;
  // block_list of the leading n0 x n0 block
  std::vector<int64_t> b0s;
  std::vector<int> szs;
  {
    int64_t i = 0;
    while (i < n0) {
      const int s = (i + 1 < n0 && t[(i + 1) * ld + i] != 0.0) ? 2 : 1;
      b0s.push_back(i);
      szs.push_back(s);
      i += s;
    }
  }
  Cx prod[2];
  for (int64_t bi = static_cast<int64_t>(b0s.size()) - 1; bi >= 0; --bi) {
    const int64_t b0 = b0s[bi];
    const int sz = szs[bi];
    const int64_t b1 = b0 + sz;
    rmat_cvec(b, t + b0 * ld + b1, sz, n0 - b1, ld, x + b1, prod, buf);
    Cx r[2];
    for (int k = 0; k < sz; ++k) r[k] = csub(rhs[b0 + k], prod[k]);
    if (sz == 1) {
      Cx piv = csub(cx(t[b0 * ld + b0]), lam);
      if (cabs_(piv) < tiny) piv = cx(tiny);
      x[b0] = cdiv(r[0], piv);
    } else {
      Cx m00 = cx(t[b0 * ld + b0]), m01 = cx(t[b0 * ld + b0 + 1]), m10 = cx(t[(b0 + 1) * ld + b0]),
         m11 = cx(t[(b0 + 1) * ld + b0 + 1]);
      m00 = csub(m00, lam);
      m11 = csub(m11, lam);
      Cx det = csub(cmul(m00, m11), cmul(m01, m10));
      if (cabs_(det) < tiny * tiny) det = cx(tiny * tiny);
      x[b0] = cdiv(csub(cmul(m11, r[0]), cmul(m01, r[1])), det);
      x[b0 + 1] = cdiv(csub(cmul(m00, r[1]), cmul(m10, r[0])), det);
    }
  }
}

}  // namespace

// schur_eigenvectors(form, indices) (schur.py:446-487): for each picked
// block (index into T's block list), the eigenvalue (vals[2k], vals[2k+1])
// and the unit eigenvector Z y as row k of vecs (nsel x zrows, complex
// interleaved).  Z is zrows x n, C-order.  0 ok, -1 bad arguments.
KLS_API int kls_schur_eigenvectors(const double* t, const double* z, int64_t n, int64_t zrows,
                                   const int64_t* picks, int64_t npick, double* vals,
                                   double* vecs, const KlsHostBlas* tbl) {
  Blas b;
  if (t == nullptr || z == nullptr || n < 0 || !load(tbl, &b) || !b.zgemv || !b.zdotu) return -1;
  std::vector<int64_t> b0s;
  std::vector<int> szs;
  block_list(t, n, b0s, szs);
  std::vector<Cx> y(n), rhs(n), buf, zc;
  for (int64_t k = 0; k < npick; ++k) {
    const int64_t blk = picks[k];
    if (blk < 0 || blk >= static_cast<int64_t>(b0s.size())) return -1;
    const int64_t b0 = b0s[blk];
    const int sz = szs[blk];
    Cx lam, head[2];
    if (sz == 1) {
      lam = cx(t[b0 * n + b0]);
      head[0] = cx(1.0);
    } else {
      const double a = t[b0 * n + b0], bb = t[b0 * n + b0 + 1], c = t[(b0 + 1) * n + b0],
                   d = t[(b0 + 1) * n + b0 + 1];
      const double half = 0.5 * (a - d);
      const double disc = half * half + bb * c;
      const double centre = 0.5 * (a + d);
      Cx p0, p1;
      if (disc >= 0.0) {
        const double r = std::sqrt(disc);
        p0 = cx(centre + r), p1 = cx(centre - r);
      } else {
        const double r = std::sqrt(-disc);
        p0 = Cx{centre + 0.0, 0.0 + r};  // centre + 1j * r
        p1 = Cx{centre - 0.0, 0.0 - r};
      }
      lam = p0.im >= 0 ? p0 : p1;
      const Cx c1[2] = {cx(bb), csub(lam, cx(a))};
      const Cx c2[2] = {csub(lam, cx(d)), cx(c)};
      const double s1 = cabs_(c1[0]) + cabs_(c1[1]);
      const double s2 = cabs_(c2[0]) + cabs_(c2[1]);
      head[0] = s1 >= s2 ? c1[0] : c2[0];
      head[1] = s1 >= s2 ? c1[1] : c2[1];
    }
    // rhs = -(T[:b0, b0:b0+sz] @ head)
    if (b0) {
      rmat_cvec(b, t + b0, b0, sz, n, head, rhs.data(), buf);
      for (int64_t i = 0; i < b0; ++i) rhs[i] = Cx{-rhs[i].re, -rhs[i].im};
    }
    back_substitute(b, t, b0, n, lam, rhs.data(), y.data(), buf);
    for (int i = 0; i < sz; ++i) y[b0 + i] = head[i];
    for (int64_t i = b0 + sz; i < n; ++i) y[i] = cx(0.0);
    // y /= np.linalg.norm(y): sqrt(y.real . y.real + y.imag . y.imag)
    const double* yd = reinterpret_cast<const double*>(y.data());
    const double sq = npdot(b, n, yd, 2, yd, 2) + npdot(b, n, yd + 1, 2, yd + 1, 2);
    const Cx nr = cx(std::sqrt(sq));
    for (int64_t i = 0; i < n; ++i) y[i] = cdiv(y[i], nr);
    // Z @ y
    Cx* out = reinterpret_cast<Cx*>(vecs) + k * zrows;
    rmat_cvec(b, z, zrows, n, n, y.data(), out, zc);
    vals[2 * k] = lam.re;
    vals[2 * k + 1] = lam.im;
  }
  return 0;
}

// hessenberg_reduce (schur.py:95-124 of this package; reference schur.py):
// H (n x n, C-order) in place, U out (n x n, C-order).
KLS_API int kls_hessenberg_reduce(double* h, double* u, int64_t n, const KlsHostBlas* tbl) {
  Blas b;
  if (h == nullptr || u == nullptr || n < 0 || !load(tbl, &b)) return -1;
  for (int64_t r = 0; r < n; ++r)
    for (int64_t c = 0; c < n; ++c) u[r * n + c] = (r == c) ? 1.0 : 0.0;
  std::vector<double> v(n), w(n);
  for (int64_t j = 0; j + 2 < n; ++j) {
    const int64_t len = n - j - 1;
    const double* col = h + (j + 1) * n + j;  // stride n
    const double tail = npdot(b, len - 1, col + n, n, col + n, n);
    const double c0 = col[0];
    if (tail == 0.0 && c0 >= 0.0) continue;
    double beta;
    if (tail == 0.0) {
      for (int64_t i = 0; i < len; ++i) v[i] = col[i * n];
      v[0] = 1.0;
      beta = 2.0;
    } else {
      const double mu = std::sqrt(c0 * c0 + tail);
      const double head = c0 <= 0.0 ? c0 - mu : -tail / (c0 + mu);
      beta = 2.0 * head * head / (tail + head * head);
      for (int64_t i = 0; i < len; ++i) v[i] = col[i * n] / head;
      v[0] = 1.0;
    }
    // w = beta * (v @ H[j+1:, :]); H[j+1:, :] -= outer(v, w)
    reflect_rows(b, h, n, v.data(), beta, j + 1, len, 0, w);
    // w = beta * (H[:, j+1:] @ v); H[:, j+1:] -= outer(w, v); the same for U
    reflect_cols(b, h, n, v.data(), beta, n, j + 1, len, w);
    reflect_cols(b, u, n, v.data(), beta, n, j + 1, len, w);
    for (int64_t r = j + 2; r < n; ++r) h[r * n + j] = 0.0;
  }
  return 0;
}

// _francis_sweeps + the final 2x2 split pass of hessenberg_real_schur
// (schur.py:206-291): T (upper Hessenberg) and Z (accumulated, usually the
// identity) in place.  Returns 0, or 1 when max_sweeps is exceeded
// (IterationLimitError).
KLS_API int kls_schur_sweeps(double* t, double* z, int64_t n, int64_t max_sweeps,
                             const KlsHostBlas* tbl) {
  Blas b;
  if (t == nullptr || z == nullptr || n < 0 || !load(tbl, &b)) return -1;
  if (n > 2 && !francis_sweeps(b, t, z, n, max_sweeps)) return 1;
  std::vector<int64_t> b0;
  std::vector<int> sz;
  std::vector<double> tmp(2 * n + 4);
  block_list(t, n, b0, sz);
  for (size_t k = 0; k < b0.size(); ++k)
    if (sz[k] == 2) split_block(b, t, z, n, b0[k], tmp);
  return 0;
}

// swap_adjacent_blocks(T, Z, i, p, q) (schur.py:294-319): 1 swapped, 0
// refused (T, Z untouched), -1 bad arguments / LAPACK error.
KLS_API int kls_schur_swap(double* t, double* z, int64_t n, int64_t i, int32_t p, int32_t q,
                           const KlsHostBlas* tbl) {
  Blas b;
  if (t == nullptr || z == nullptr || p < 1 || p > 2 || q < 1 || q > 2 || i < 0 ||
      i + p + q > n || !load(tbl, &b))
    return -1;
  std::vector<double> tmp(4 * n + 16);
  return swap_blocks(b, t, z, n, i, p, q, tmp);
}

// move_blocks_front(form, selected) (schur.py:346-371): flags, one per
// diagonal block of T in order; returns the total size moved, or -1 when
// the flag count does not match the block count (DimensionError).
KLS_API int64_t kls_schur_move_front(double* t, double* z, int64_t n, const uint8_t* selected,
                                     int64_t nsel, const KlsHostBlas* tbl) {
  Blas b;
  if (t == nullptr || z == nullptr || n < 0 || !load(tbl, &b)) return -2;
  std::vector<int64_t> b0;
  std::vector<int> sz;
  block_list(t, n, b0, sz);
  if (static_cast<int64_t>(b0.size()) != nsel) return -1;
  std::vector<uint8_t> flags(selected, selected + nsel);
  std::vector<double> tmp(4 * n + 16);
  int64_t front = 0, moved = 0;
  for (int64_t blk = 0; blk < nsel; ++blk) {
    if (!flags[blk]) continue;
    int64_t cur = blk;
    while (cur > front) {
      const int64_t s0 = b0[cur - 1];
      const int z0 = sz[cur - 1], z1 = sz[cur];
      const int r = swap_blocks(b, t, z, n, s0, z0, z1, tmp);
      if (r < 0) return -2;
      if (r == 0) break;
      b0[cur - 1] = s0, sz[cur - 1] = z1;
      b0[cur] = s0 + z1, sz[cur] = z0;
      std::swap(flags[cur - 1], flags[cur]);
      cur -= 1;
    }
    if (cur == front) {
      moved += sz[front];
      front += 1;
    }
  }
  return moved;
}
