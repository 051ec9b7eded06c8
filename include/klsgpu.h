/*
 * klsgpu.h — C-ABI of libklsgpu.so, the sm_100a kernels behind the
 * DCGS2 / CGS2 Arnoldi-QR hot path of arXiv 2104.01253.
 *
 * Every entry point takes plain device pointers, sizes, leading dimensions
 * and a cudaStream_t passed as void*.  Nothing allocates: workspaces are
 * caller-owned (size them with kls_workspace_bytes and zero them once).
 * Return value: 0 on success, <0 on error (KLS_EINVAL bad argument,
 * KLS_ECUDA CUDA error, KLS_ENOSPC workspace too small); the message is in
 * kls_last_error() (thread-local).  Numerical breakdowns are not errors at
 * this level: the host decides them from the reduced scalars and raises the
 * reference's exceptions (errors.py:4-39).
 *
 * Layout: a basis block Q is column-major with leading dimension ldq (even;
 * the Python host pads it to a multiple of 32 doubles).  Vectors are fp64
 * arrays of m rows, 16-byte aligned.  Reductions are deterministic (fixed
 * summation order, no fp64 atomics) AND independent of the number of ranks
 * the rows are split over: they follow the fixed segment tree of KlsSegs
 * below, so 1, 2, 3, 4, 6 or 8 GPUs give bitwise-identical results.
 *
 * Each declaration cites the reference interface it replaces
 * (/root/reference/pkg/src/kls/<file>:<line>).
 */
#ifndef KLSGPU_H
#define KLSGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KLS_OK 0
#define KLS_EINVAL (-1)
#define KLS_ECUDA (-2)
#define KLS_ENOSPC (-3)

/* Library ABI version (1). */
int kls_version(void);
/* Message of the last failing call on this thread. */
const char* kls_last_error(void);
/* SM count of the current device (grid sizing). */
int kls_device_sm_count(void);
/* cudaStreamSynchronize(stream): the one host wait of a DCGS2 step. */
int kls_stream_sync(void* stream);
/* Device address of page-locked host memory, so a reduction can deposit its
 * 2j+3 scalars straight into a pinned host buffer (no D2H copy call). */
int kls_host_device_ptr(void* host, void** dev);

/* Bytes of reduction workspace that cover any call with <= kmax basis
 * columns on the current device.  Zero it once before first use; every
 * reducing kernel leaves its tickets at zero again. */
size_t kls_workspace_bytes(int64_t m, int32_t kmax);

/* ---- rank-count-independent reductions -----------------------------------
 * The global rows [0, m) are cut into 24 segments at multiples of `unit`
 * rows (64 for CSR / dense / QR blocks, a stencil's x-plane — even); rank r
 * of `world` (1 <= world <= 24) owns segments [r*24/world, (r+1)*24/world)
 * and therefore rows kls_seg_rows(); its local m must equal that range.
 * Every reduction sums segments over one fixed tree, so its result does not
 * depend on world.  With world > 1 a reduction that is not fused with a
 * peer exchange writes this rank's EXPORTED tree nodes instead of the
 * result: out[e * xstride + o] for its e-th exported node (<= 8 nodes;
 * xstride = the call's output count unless stated), which
 * kls_peer_seg_combine or (after an all_gather) kls_seg_combine turn into
 * the global values.  NULL KlsSegs = one rank holding all m rows, unit 64.
 * The reference has one process and numpy sums (kernels.py:44-60); this is
 * the layout its MPI_Allreduce becomes here. */
typedef struct KlsSegs {
  int64_t m;     /* global rows */
  int64_t unit;  /* partition unit (rows, even) */
  int32_t world; /* ranks */
  int32_t rank;  /* this rank */
} KlsSegs;
/* This rank's global rows [lo, hi). */
int kls_seg_rows(const KlsSegs* s, int64_t* lo, int64_t* hi);
/* The tree nodes rank exports, left to right (ids[<= 8]); returns the count. */
int kls_seg_exports(int32_t rank, int32_t world, int32_t* ids);
/* blocks = [world][8][stride] gathered export blocks -> out[0:nout]. */
int kls_seg_combine(const double* blocks, int32_t nout, int64_t stride, int32_t world, double* out,
                    void* stream);

/* Fused block inner products — kernels.mv_trans_mv (kernels.py:44-60):
 *   out = [Q(:, 0:k), bext]^T [x0 (, x1)]      column-major,
 *         (k + (bext != NULL)) rows x nx columns (nx = 1 or 2),
 *   then out[rows*nx] = x_last . x_last when xnorm != 0.
 * bext == NULL drops the extra left column; k == 0 is allowed (the empty
 * basis block still reduces, kernels.py:5-9).  One pass over Q. */
int kls_mv_trans_mv(const double* Q, int64_t ldq, int64_t m, int32_t k, const double* bext,
                    const double* x0, const double* x1, int32_t nx, int32_t xnorm, double* out,
                    const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream);

/* The single fused reduction of a DCGS2 Arnoldi step — replaces
 *   g = mv_trans_mv(np.hstack([Q, w]), np.column_stack([w, aw]))
 * (arnoldi.py:362-370) plus the guard norm ||aw|| (arnoldi.py:414):
 *   out[0:j]   = c = Q^T w      out[j]     = beta  = w.w
 *   out[j+1:2j+1] = s = Q^T aw  out[2j+1]  = s_piv = w.aw
 *   out[2j+2]  = aw.aw
 * 2j+3 doubles: the payload of the one allreduce per step. */
int kls_gram_dcgs2(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                   const double* aw, double* out, const KlsSegs* segs, void* ws, size_t ws_bytes,
                   void* stream);

/* Fused DCGS2 update — the two MvTimesMatAddMv of a step
 * (arnoldi.py:389-391 and 415-420; QR form ortho.py:371-375, 396-398):
 *   u = w - Q(:,0:j) c;  Q(:, j) = u / alpha;
 *   w = (divide ? aw / alpha : aw) - (Q(:,0:j) t(0:j) + Q(:,j) t_j)
 * coef (device) = [c(0:j), t(0:j+1)], 2j+1 doubles.  One pass over Q.
 * segs: the rows' layout (NULL: one rank) -- only its global row count is
 * used, to pick the same kernel (the same per-row arithmetic) on every rank. */
int kls_dcgs2_update(double* Q, int64_t ldq, int64_t m, int32_t j, double* w, const double* aw,
                     const double* coef, double alpha, int32_t divide, const KlsSegs* segs,
                     void* stream);

/* kls_dcgs2_update with the 2j+1 coefficients in HOST memory: they are
 * carried in the kernel launch (2j+1 <= 2048), so a step needs no H2D copy. */
int kls_dcgs2_update_host(double* Q, int64_t ldq, int64_t m, int32_t j, double* w,
                          const double* aw, const double* coef_host, double alpha, int32_t divide,
                          const KlsSegs* segs, void* stream);

/* Device-side scalar step (arnoldi.py:379-400): from g = [c, beta, s, s_piv,
 * aw.aw] (device) write coef = [c, s/alpha, t_piv, alpha] (device, 2j+2;
 * qr != 0: the QR form of ortho.py:369) and copy g to gout (mapped host
 * memory or NULL) — lets the update be queued one step ahead of the host. */
int kls_dcgs2_scalars(const double* g, int32_t j, int32_t qr, double* coef, double* gout,
                      void* stream);
/* kls_dcgs2_update with coef_alpha = [c, t, alpha] on the device (from
 * kls_dcgs2_scalars), writing w' to w_out and leaving w intact (a
 * speculative step can be discarded). */
int kls_dcgs2_update_dev(double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                         double* w_out, const double* aw, const double* coef_alpha,
                         int32_t divide, const KlsSegs* segs, void* stream);

/* Y(:,0:l) <- scale*Y + sign*B(:,0:k) S — kernels.mv_times_mat_add_mv
 * (kernels.py:63-84) for l = 1 or 2; S is k x l column-major on the device.
 * nrm_out (optional, device) receives ||Y(:, l-1)||^2 of the result, fusing
 * the norm2 that follows a projection (ortho.py:153-154, arnoldi.py:433-434). */
int kls_mv_times_mat_add_mv(double* Y, int64_t ldy, int64_t m, int32_t l, const double* B,
                            int64_t ldb, int32_t k, const double* S, double sign, double scale,
                            double* nrm_out, const KlsSegs* segs, void* ws, size_t ws_bytes,
                            void* stream);
/* Same with S in HOST memory (k*l <= 2048), carried in the launch. */
int kls_mv_times_mat_add_mv_host(double* Y, int64_t ldy, int64_t m, int32_t l, const double* B,
                                 int64_t ldb, int32_t k, const double* S_host, double sign,
                                 double scale, double* nrm_out, const KlsSegs* segs, void* ws,
                                 size_t ws_bytes, void* stream);

/* CGS2 comparator, fused first update + second projection of
 * Cgs2State.push (reference ortho.py:148-151, i.e. MvTimesMatAddMv followed
 * by MvTransMv, kernels.py:40-84): v <- v - Q(:,0:k) s in place, then
 * out[0:k] = Q^T v and, when xnorm != 0, out[k] = v.v.  The chunk's Q rows
 * are re-read from L2, so the pair costs one HBM pass over Q.  1 <= k <= 2048;
 * s is host memory (carried in the launch) when s_on_host != 0, else device. */
int kls_project_gram(const double* Q, int64_t ldq, int64_t m, int32_t k, double* v,
                     const double* s, int32_t s_on_host, int32_t xnorm, double* out,
                     const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream);

/* y = A x for CSR rows (int64 row pointer, int32 columns, fp64 values),
 * bit-identical to CsrMatrix.matvec (problems.py:127-136): products, then
 * numpy's reduceat/pairwise summation order per row. */
int kls_csr_spmv(const int64_t* rowptr, const int32_t* col, const double* val, int64_t nrows,
                 const double* x, double* y, void* stream);

/* ELL copy of a CSR block with <= width (<= 8) entries per row: entry k of
 * row i at k*ld + i (coalesced streams); elen[i] = row length. */
int kls_csr_to_ell(const int64_t* rowptr, const int32_t* col, const double* val, int64_t nrows,
                   int32_t width, int64_t ld, int32_t* ecol, double* eval, uint8_t* elen,
                   void* stream);
/* y = A x from that layout, bit-identical to kls_csr_spmv (same per-row
 * entry order, same reduceat summation). */
int kls_ell_spmv(const int32_t* ecol, const double* eval, const uint8_t* elen, int32_t width,
                 int64_t nrows, int64_t ld, const double* x, double* y, void* stream);
/* GMRES backward-error norms fused with the ELL product (gmres.py:46-60):
 * out = [||b - A x||^2, ||x||^2, ||b||^2] for a one-rank ELL operator; A x is
 * formed bit-identically to kls_ell_spmv and not stored. */
int kls_ell_resid_norms(const int32_t* ecol, const double* eval, const uint8_t* elen,
                        int32_t width, int64_t nrows, int64_t ld, const double* x,
                        const double* b, double* out, const KlsSegs* segs, void* ws,
                        size_t ws_bytes, void* stream);

/* y2 = A x2 (bit-identical to kls_ell_spmv) and the norms of
 * kls_ell_resid_norms for (x, b) (bit-identical) in one pass over the
 * entries of a one-rank ELL operator. */
int kls_ell_apply_resid_norms(const int32_t* ecol, const double* eval, const uint8_t* elen,
                              int32_t width, int64_t nrows, int64_t ld, const double* x2,
                              double* y2, const double* x, const double* b, double* out,
                              const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream);

/* Matrix-free 7-point Laplacian, bit-identical to StencilLaplace3D._matvec
 * (problems.py:296-305) on nx local x-planes of a (.., ny, nz) grid; x_lo /
 * x_hi are the neighbouring planes of other ranks (NULL at the boundary). */
int kls_stencil7(const double* x, const double* x_lo, const double* x_hi, double* y, int64_t nx,
                 int64_t ny, int64_t nz, void* stream);

/* y = A x for a row-major dense A (DenseOperator._matvec, problems.py:76-77). */
int kls_dense_gemv(const double* a, int64_t lda, int64_t n, const double* x, double* y,
                   void* stream);

/* y = x / alpha (mode 0, the normalisations u / alpha of arnoldi.py:391,453,
 * ortho.py:136,158,398) or y = x * alpha (mode 1). */
int kls_scale(const double* x, double* y, int64_t n, double alpha, int32_t mode, void* stream);

/* out = a - b (restart residual b - A x, gmres.py:151). */
int kls_sub(const double* a, const double* b, double* out, int64_t n, void* stream);

/* Backward-error norms in one pass (gmres.backward_error, gmres.py:46-60):
 * out = [||b - ax||^2, ||x||^2, ||b||^2] (device). */
int kls_resid_norms(const double* b, const double* ax, const double* x, int64_t n, double* out,
                    const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream);

/* V(:, 0:k) <- V(:, 0:k) Z in place, Z k x k column-major on the device —
 * the Krylov-Schur basis rotation v_mat[:, nlock:k] @ Z (eig.py:237). */
int kls_tsgemm_inplace(double* V, int64_t ldv, int64_t m, int32_t k, const double* Z,
                       void* stream);
/* V(:, 0:p) <- V(:, 0:k) Z(:, 0:p) in place, Z k x p column-major on the
 * device (eig.py:237 keeps the first p columns of V Z).  Register-blocked;
 * V 16-byte aligned, even ldv. */
int kls_tsgemm_inplace_cols(double* V, int64_t ldv, int64_t m, int32_t k, int32_t p,
                            const double* Z, void* stream);

/* ---- device-side operator construction -------------------
 * CSR of a row block [row_lo, row_lo + nrows) built directly in HBM, entry
 * for entry identical to the reference's host assembly; columns are stored
 * relative to the global row col_base (the rank's extended-vector origin);
 * rowptr (nrows + 1 entries) starts at 0.  *_nnz give the block's size. */
int64_t kls_lap7_nnz(int64_t nx, int64_t ny, int64_t nz, int64_t row_lo, int64_t row_hi);
/* StencilLaplace3D.to_csr (problems.py:307-331). */
int kls_build_lap7_csr(int64_t nx, int64_t ny, int64_t nz, int64_t row_lo, int64_t nrows,
                       int64_t col_base, int64_t* rowptr, int32_t* col, double* val, void* stream);
int64_t kls_mant5_nnz(int64_t k, int64_t row_lo, int64_t row_hi);
/* manteuffel_build (problems.py:208-245); diff = 1/h^2, conv = beta/(2h). */
int kls_build_mant5_csr(int64_t k, int64_t row_lo, int64_t nrows, int64_t col_base, double diff,
                        double conv, int64_t* rowptr, int32_t* col, double* val, void* stream);
/* Banded random operator of order m (config 5's Arnoldi variant, SURVEY.md
 * §8d "random banded operator, bandwidth <= 1e3 so halos stay local"): row i
 * holds d entries, one per equal slice of [max(0, i-band), min(m, i+band+1)),
 * hashed column and value in [-1, 1) from (seed, i, slice) -- the host
 * restatement oracle.band_random_coo + kls.CsrMatrix.from_coo
 * (problems.py:99-117) gives the same CSR bit for bit.  d <= 2 band + 1. */
int kls_build_band_csr(int64_t m, int64_t band, int32_t d, uint64_t seed, int64_t row_lo,
                       int64_t nrows, int64_t col_base, int64_t* rowptr, int32_t* col,
                       double* val, void* stream);

/* ---- one-GPU step plan ------------------------------------------------------
 * The DCGS2 lookahead's per-step launches in one host call
 * (paper_2104_01253_b200/arnoldi.py _step_ahead): update of step j (w ->
 * w_out, column j of Q; coefficients from the previous scalar step in cdev),
 * the operator (x_out = w_out's operand address -> aw_out), and, when gram
 * != 0, the fused Gram + scalar step of step j+1 into gdev / cdev /
 * gout[slot], then event[slot] is recorded. */
enum { KLS_OP_ELL = 1, KLS_OP_CSR = 2, KLS_OP_STENCIL7 = 3, KLS_OP_DENSE = 4 };
typedef struct {
  int32_t kind;   /* KLS_OP_* */
  int32_t width;  /* ELL: entries per row */
  int64_t m;      /* rows */
  int64_t n0;     /* ELL: ld; stencil: nx; dense: lda */
  int64_t n1;     /* stencil: ny */
  int64_t n2;     /* stencil: nz */
  const void* p0; /* ELL: ecol; CSR: rowptr; dense: a */
  const void* p1; /* ELL: eval; CSR: col */
  const void* p2; /* ELL: elen; CSR: val */
} KlsOpDesc;
typedef struct {
  double* Q;
  int64_t ldq;
  int64_t m;
  KlsSegs segs;   /* the rows' layout (world 1 here) */
  double* gdev;
  double* cdev;
  double* gout[2];
  void* ws;
  size_t ws_bytes;
  void* stream;
  void* event[2];
  int32_t divide; /* 1: Arnoldi form, 0: QR form */
  int32_t qr;     /* scalar step in QR form */
  KlsOpDesc op;
} KlsStepPlan;
int kls_dcgs2_queue_step(const KlsStepPlan* plan, int32_t j, const double* w, double* w_out,
                         const double* x_out, const double* aw, double* aw_out, int32_t slot,
                         int32_t gram);
typedef struct {
  const KlsStepPlan* plan;
  double* w[2];          /* local rows of the two pending-vector buffers */
  const double* wx[2];   /* their operand addresses for the operator */
  double* aw[2];         /* their images */
  const double* gslot[2];/* host views of the mapped result slots (plan->gout) */
  double* h;             /* C-order Hessenberg buffer, row stride ldh */
  int64_t ldh;
  double* k;             /* K: in for step j0, out after the last step (capacity) */
  double* scratch;       /* 2 * capacity doubles */
  void* ddot;            /* cblas_ddot / cblas_dgemv for kls_dcgs2_host_step */
  void* dgemv;
  int64_t m;             /* global rows (guards) */
  int32_t capacity;
} KlsRunState;
/* Up to nsteps DCGS2 lookahead steps in one call (one GPU): per step
 * kls_dcgs2_queue_step, a wait on the step's scalars and
 * kls_dcgs2_host_step; stops at a breakdown.  See plan.cu for io. */
int kls_dcgs2_run(const KlsRunState* s, int32_t j0, int32_t nsteps, int32_t cur, int32_t slot,
                  double* io);
/* GMRES's per-column backward error (gmres.py:166-172) of an earlier column
 * riding on a lookahead step: xj = x + Q(:, 0:q) y (y: q HOST doubles, read
 * during the call) and out = [||b - A xj||^2, ||xj||^2, ||b||^2] (device). */
typedef struct {
  const double* x;
  double* xj;
  int32_t q;
  const double* y;
  const double* b;
  double* out;
} KlsBeCol;
/* kls_dcgs2_queue_step (gram != 0 required for the Gram part as there) with
 * the backward-error column fused into the update and the ELL product: the
 * same bits as the separate launches, without their passes over Q and A. */
int kls_dcgs2_queue_step_be(const KlsStepPlan* plan, int32_t j, const double* w, double* w_out,
                            const double* x_out, const double* aw, double* aw_out, int32_t slot,
                            int32_t gram, const KlsBeCol* be);
int kls_event_create(void** ev);
int kls_event_destroy(void* ev);
int kls_event_record(void* ev, void* stream);
int kls_event_sync(void* ev);

/* ---- cross-GPU exchange over NVLink peer memory ---------------------------
 * Symmetric buffers (same layout on every rank, mapped into every peer) of
 * kls_peer_buffer_bytes(cap) bytes; bufs[r] is rank r's buffer as seen from
 * this GPU.  All spins time out after 20 s and set *err instead of hanging. */
size_t kls_peer_buffer_bytes(int32_t cap);

/* Peer buffers for hosts without a collective allocator (the reference's
 * mpi4py-style SPMD launch; SURVEY.md §8b kls_comm_init): allocate and zero
 * this rank's buffer and get its IPC handle (kls_ipc_handle_bytes() bytes),
 * exchange handles over the caller's bootstrap, open every peer's handle,
 * and pass the resulting pointer table as `bufs` below (own rank: its own
 * buffer).  Close peers and free the own buffer when done. */
size_t kls_ipc_handle_bytes(void);
int kls_peer_buffer_alloc(size_t bytes, void** buf, void* handle);
int kls_peer_buffer_open(const void* handle, void** peer_buf);
int kls_peer_buffer_close(void* peer_buf);
int kls_peer_buffer_free(void* buf);

/* A reduction's global combine (ledger site
 * kernels.py:57-59) as a one-shot NVLink exchange: src holds this rank's
 * exported node values of nv outputs ([e][nv], as a reduction with world > 1
 * writes them); every rank publishes them, and all evaluate the fixed
 * segment tree into out (device or mapped host memory) — bitwise identical
 * on all ranks and to a one-rank run.  epoch: +1 per call, same on all
 * ranks; 8 * nv <= cap. */
int kls_peer_seg_combine(const double* src, int32_t nv, double* out, void* const* bufs,
                         int32_t rank, int32_t world, int32_t cap, uint64_t epoch, int* err,
                         void* stream);

/* kls_gram_dcgs2 with the step's device scalar arithmetic (kls_dcgs2_scalars)
 * fused into the kernel's last CTA: out <- g (2j+3), coef <- [c, s/alpha
 * (QR: s), t_piv, alpha] (2j+2), gout <- g (mapped host memory or NULL).
 * j <= 1024.  One launch per step for arnoldi.py:362-400 / ortho.py:378-399. */
int kls_gram_dcgs2_step(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                        const double* aw, double* out, double* coef, double* gout, int32_t qr,
                        const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream);

/* Host half of a DCGS2 Arnoldi step (arnoldi.py:367-420) in C++: guards,
 * Pythagorean alpha, Stephen's-trick t_piv, Hessenberg column j-1 and the
 * correction K, reproducing numpy's arithmetic bit for bit when ddot / dgemv
 * are numpy's own cblas_ddot / cblas_dgemv (ILP64).  h: C-order Hessenberg
 * buffer with row stride ldh.  Returns 0 (t_full, k_next: j+1 values;
 * res = [alpha, vscale]), 1 happy breakdown, 2 Pythagorean breakdown. */
int kls_dcgs2_host_step(const double* g, int32_t j, int64_t m, double wscale,
                        const double* k_prev, double* h, int64_t ldh, double* t_full,
                        double* k_next, double* res, void* ddot, void* dgemv);

/* Host real-Schur services for Krylov-Schur restarts (schur.py:84-410) in
 * C++, bit for bit with the reference's numpy arithmetic when the table
 * holds numpy's own ILP64 OpenBLAS entry points (cblas_ddot, cblas_dgemv,
 * cblas_dgemm, dgesv_, dgeqrf_, dorgqr_).  Matrices are C-order n x n. */
typedef struct KlsHostBlas {
  void* ddot;
  void* dgemv;
  void* dgemm;
  void* dgesv;
  void* dgeqrf;
  void* dorgqr;
  void* zgemv;     /* cblas_zgemv, cblas_zdotu_sub (eigenvectors) */
  void* zdotu_sub;
} KlsHostBlas;
/* hessenberg_reduce (schur.py:84-114): H in place, U out.  0 / -1. */
int kls_hessenberg_reduce(double* h, double* u, int64_t n, const KlsHostBlas* blas);
/* Francis double-shift sweeps + the final 2x2 split pass of
 * hessenberg_real_schur (schur.py:176-290) on T, accumulating into Z.
 * 0 ok, 1 sweep limit exceeded (IterationLimitError), -1 bad arguments. */
int kls_schur_sweeps(double* t, double* z, int64_t n, int64_t max_sweeps,
                     const KlsHostBlas* blas);
/* schur_eigenvectors (schur.py:446-487) for the picked blocks: vals
 * (npick complex, interleaved), vecs (npick rows of zrows complex: Z y). */
int kls_schur_eigenvectors(const double* t, const double* z, int64_t n, int64_t zrows,
                           const int64_t* picks, int64_t npick, double* vals, double* vecs,
                           const KlsHostBlas* blas);
/* swap_adjacent_blocks (schur.py:305-340): 1 swapped, 0 refused. */
int kls_schur_swap(double* t, double* z, int64_t n, int64_t i, int32_t p, int32_t q,
                   const KlsHostBlas* blas);
/* move_blocks_front (schur.py:378-410): returns the size moved; -1 when nsel
 * differs from the block count (DimensionError), -2 on other errors. */
int64_t kls_schur_move_front(double* t, double* z, int64_t n, const uint8_t* selected,
                             int64_t nsel, const KlsHostBlas* blas);

/* kls_gram_dcgs2 fused with the step's global reduction: the finishing CTA
 * publishes this rank's exported tree nodes over NVLink peer memory and
 * evaluates the fixed segment tree — compute and collective in one launch
 * (8 (2 min(j, 256) + 5) <= cap; j > 256 runs as ceil(j / 256) column
 * panels that use epochs epoch, epoch + 1, ...); segs->world / rank must
 * match bufs. */
int kls_gram_dcgs2_peer(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                        const double* aw, double* out, const KlsSegs* segs, void* ws,
                        size_t ws_bytes, void* const* bufs, int32_t rank, int32_t world,
                        int32_t cap, uint64_t epoch, int* err, void* stream);

/* kls_gram_dcgs2_step fused with the peer allreduce: Gram pass, the step's
 * one global reduction and the scalar step in a single launch. */
int kls_gram_dcgs2_peer_step(const double* Q, int64_t ldq, int64_t m, int32_t j,
                             const double* w, const double* aw, double* out, double* coef,
                             double* gout, int32_t qr, const KlsSegs* segs, void* ws,
                             size_t ws_bytes, void* const* bufs, int32_t rank, int32_t world,
                             int32_t cap, uint64_t epoch, int* err, void* stream);

/* Raise this rank's halo flag (= epoch) in the buffers of the ranks set in
 * target_mask, ordered after all prior work on the stream. */
int kls_peer_signal(void* const* bufs, int32_t rank, int32_t world, int32_t target_mask,
                    uint64_t epoch, void* stream);

/* kls_stencil7 reading the neighbouring x-planes directly from peer memory
 * (x_lo / x_hi peer-mapped, NULL at the physical boundary) once the lower /
 * upper neighbour's halo flag in mybuf reaches epoch — the halo exchange of
 * the row-sharded operator (problems.py:296-305) fused into the apply. */
int kls_stencil7_peer(const double* x, const double* x_lo, const double* x_hi, double* y,
                      int64_t nx, int64_t ny, int64_t nz, void* mybuf, int32_t rank,
                      uint64_t epoch, int* err, void* stream);

/* kls_ell_spmv with the row block's halo columns read straight from the
 * neighbouring ranks' vectors over NVLink (the CSR operator's halo exchange,
 * problems.py:127-136 across ranks, fused into the apply): x_lo = the lower
 * neighbour's last nlo rows (peer-mapped), x_hi = the upper neighbour's first
 * rows (peer-mapped), NULL when absent.  Rows [b_lo, nrows - b_hi) touch only
 * owned columns and run first without waiting; the boundary rows wait for
 * this rank's halo flags from lo_rank / hi_rank (in mybuf) to reach epoch. */
int kls_ell_spmv_peer(const int32_t* ecol, const double* eval, const uint8_t* elen, int32_t width,
                      int64_t nrows, int64_t ld, const double* x, const double* x_lo, int64_t nlo,
                      const double* x_hi, double* y, int64_t b_lo, int64_t b_hi, void* mybuf,
                      int32_t lo_rank, int32_t hi_rank, uint64_t epoch, int* err, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KLSGPU_H */
