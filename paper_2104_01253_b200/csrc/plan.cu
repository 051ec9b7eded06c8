// Per-step launch plan of the one-GPU DCGS2 lookahead (arnoldi.py's
// _step_ahead): one host call queues the fused update of step j, the
// operator on its output and the Gram pass (+ scalar step) of step j + 1,
// and records the step's completion event — instead of three Python-level
// launches and a torch event.  At latency-bound sizes (config 1, GMRES and
// Krylov-Schur tails) that is the difference between a host-bound and a
// GPU-bound step.  Composes the public entry points, so the kernels and
// their results are exactly those of the launch-by-launch path.
#include "klsgpu.h"
#include "common.cuh"

using namespace kls;

namespace kls {
int gram_dcgs2_step_chain(const double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                          const double* aw, double* out, double* coef, double* gout, int32_t qr,
                          const KlsSegs* segs, void* ws, size_t ws_bytes, void* stream);  // gram.cu
int dcgs2_update_dev_comb(double* Q, int64_t ldq, int64_t m, int32_t j, const double* w,
                          double* w_out, const double* aw, const double* coef_alpha,
                          const KlsSegs* segs, void* stream, const double* x, double* xout,
                          int32_t q, const double* y);  // update.cu
}

static int apply_op(const KlsOpDesc* op, const double* x, double* y, void* stream) {
  switch (op->kind) {
    case KLS_OP_ELL:
      return kls_ell_spmv(static_cast<const int32_t*>(op->p0), static_cast<const double*>(op->p1),
                          static_cast<const uint8_t*>(op->p2), op->width, op->m, op->n0, x, y,
                          stream);
    case KLS_OP_CSR:
      return kls_csr_spmv(static_cast<const int64_t*>(op->p0), static_cast<const int32_t*>(op->p1),
                          static_cast<const double*>(op->p2), op->m, x, y, stream);
    case KLS_OP_STENCIL7:
      return kls_stencil7(x, nullptr, nullptr, y, op->n0, op->n1, op->n2, stream);
    case KLS_OP_DENSE:
      return kls_dense_gemv(static_cast<const double*>(op->p0), op->n0, op->m, x, y, stream);
    default:
      return fail(KLS_EINVAL, "step plan: unknown operator kind %d", op->kind);
  }
}

KLS_API int kls_event_create(void** ev) {
  cudaEvent_t e;
  const cudaError_t rc = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (rc != cudaSuccess) return fail(KLS_ECUDA, "event create: %s", cudaGetErrorString(rc));
  *ev = e;
  return KLS_OK;
}

KLS_API int kls_event_destroy(void* ev) {
  const cudaError_t rc = cudaEventDestroy(static_cast<cudaEvent_t>(ev));
  return rc == cudaSuccess ? KLS_OK : fail(KLS_ECUDA, "event destroy: %s", cudaGetErrorString(rc));
}

KLS_API int kls_event_record(void* ev, void* stream) {
  const cudaError_t rc = cudaEventRecord(static_cast<cudaEvent_t>(ev), static_cast<cudaStream_t>(stream));
  return rc == cudaSuccess ? KLS_OK : fail(KLS_ECUDA, "event record: %s", cudaGetErrorString(rc));
}

KLS_API int kls_event_sync(void* ev) {
  const cudaError_t rc = cudaEventSynchronize(static_cast<cudaEvent_t>(ev));
  return rc == cudaSuccess ? KLS_OK : fail(KLS_ECUDA, "event sync: %s", cudaGetErrorString(rc));
}

KLS_API int kls_dcgs2_queue_step(const KlsStepPlan* p, int32_t j, const double* w, double* w_out,
                                 const double* x_out, const double* aw, double* aw_out,
                                 int32_t slot, int32_t gram) {
  if (p == nullptr || slot < 0 || slot > 1) return fail(KLS_EINVAL, "queue_step: bad plan or slot");
  int rc = kls_dcgs2_update_dev(p->Q, p->ldq, p->m, j, w, w_out, aw, p->cdev, p->divide,
                                &p->segs, p->stream);
  if (rc) return rc;
  rc = apply_op(&p->op, x_out, aw_out, p->stream);
  if (rc) return rc;
  if (gram) {
    rc = gram_dcgs2_step_chain(p->Q, p->ldq, p->m, j + 1, w_out, aw_out, p->gdev, p->cdev,
                             p->gout[slot], p->qr, &p->segs, p->ws, p->ws_bytes, p->stream);
    if (rc) return rc;
    rc = kls_event_record(p->event[slot], p->stream);
  }
  return rc;
}


// kls_dcgs2_queue_step with GMRES's backward-error column of an earlier
// step riding on it (gmres.py:166-172): the update also forms
// be->xj = be->x + Q(:, 0:q) y from the Q tiles it streams, and on an ELL
// operator the product of w_out and the norms [||b - A xj||^2, ||xj||^2,
// ||b||^2] -> be->out are one pass over the entries.  Every value is
// bit-identical to the separate launches (add_combination, the apply,
// kls_ell_resid_norms); the column's two extra passes over Q and A go away.
KLS_API int kls_dcgs2_queue_step_be(const KlsStepPlan* p, int32_t j, const double* w,
                                    double* w_out, const double* x_out, const double* aw,
                                    double* aw_out, int32_t slot, int32_t gram,
                                    const KlsBeCol* be) {
  if (p == nullptr || be == nullptr || slot < 0 || slot > 1)
    return fail(KLS_EINVAL, "queue_step_be: bad arguments");
  if (p->op.kind != KLS_OP_ELL)
    return fail(KLS_EINVAL, "queue_step_be: needs an ELL operator");
  int rc = dcgs2_update_dev_comb(p->Q, p->ldq, p->m, j, w, w_out, aw, p->cdev, &p->segs,
                                 p->stream, be->x, be->xj, be->q, be->y);
  if (rc) return rc;
  rc = kls_ell_apply_resid_norms(static_cast<const int32_t*>(p->op.p0),
                                 static_cast<const double*>(p->op.p1),
                                 static_cast<const uint8_t*>(p->op.p2), p->op.width, p->op.m,
                                 p->op.n0, x_out, aw_out, be->xj, be->b, be->out, &p->segs, p->ws,
                                 p->ws_bytes, p->stream);
  if (rc) return rc;
  if (gram) {
    rc = gram_dcgs2_step_chain(p->Q, p->ldq, p->m, j + 1, w_out, aw_out, p->gdev, p->cdev,
                             p->gout[slot], p->qr, &p->segs, p->ws, p->ws_bytes, p->stream);
    if (rc) return rc;
    rc = kls_event_record(p->event[slot], p->stream);
  }
  return rc;
}

// The lookahead loop itself (arnoldi.py:349-423 per step, _step_ahead's
// order): per step one queue_step, one wait on the step's scalars, the C++
// host step; stops after nsteps, at a breakdown, or when the next Gram would
// not fit the basis.  io: [0] wscale (in/out), [1] alpha of the first
// completed step, [2] steps completed, [3] status (0 / 1 happy / 2
// Pythagorean), [4] j of the stopping step, [5] slot of the queued next Gram
// (-1: none), [6] buffer index of the pending vector.
KLS_API int kls_dcgs2_run(const KlsRunState* s, int32_t j0, int32_t nsteps, int32_t cur,
                          int32_t slot, double* io) {
  if (s == nullptr || io == nullptr || cur < 0 || cur > 1 || slot < 0 || slot > 1)
    return fail(KLS_EINVAL, "dcgs2_run: bad arguments");
  double wscale = io[0];
  double* t_full = s->scratch;
  double* k_next = s->scratch + s->capacity;
  double res[2];
  int32_t done = 0, status = 0, jstop = j0;
  for (int32_t t = 0; t < nsteps; ++t) {
    const int32_t j = j0 + t;
    const int32_t nxt = j + 2 < s->capacity ? 1 - slot : -1;
    int rc = kls_dcgs2_queue_step(s->plan, j, s->w[cur], s->w[1 - cur], s->wx[1 - cur],
                                  s->aw[cur], s->aw[1 - cur], nxt >= 0 ? nxt : 0, nxt >= 0);
    if (rc) return rc;
    rc = kls_event_sync(s->plan->event[slot]);
    if (rc) return rc;
    const int st = kls_dcgs2_host_step(s->gslot[slot], j, s->m, wscale, s->k, s->h, s->ldh,
                                       t_full, k_next, res, s->ddot, s->dgemv);
    if (st < 0) return fail(KLS_EINVAL, "dcgs2_run: host step arguments");
    jstop = j;
    if (st != 0) {
      status = st;
      break;
    }
    if (done == 0) io[1] = res[0];
    for (int32_t i = 0; i <= j; ++i) s->k[i] = k_next[i];
    wscale = res[1];
    ++done;
    cur = 1 - cur;
    slot = nxt;
    if (nxt < 0) break;  // no Gram queued for j + 1: the caller finishes
  }
  io[0] = wscale;
  io[2] = done;
  io[3] = status;
  io[4] = jstop;
  io[5] = slot;
  io[6] = cur;
  return KLS_OK;
}
