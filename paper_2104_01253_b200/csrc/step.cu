// Device-side scalar step of DCGS2 (the arithmetic of arnoldi.py:379-400,
// ortho.py:387-399) so the update kernel can be queued before the host has
// looked at the step's reduced scalars (a one-step lookahead: the host's
// numpy bookkeeping of H / K and the reference's guards then run while the
// GPU already streams the update, the operator and the next Gram pass).
//
// From g = [c(0:j), beta, s(0:j), s_piv, aw.aw] (kls_gram_dcgs2) it writes
//   coef = [c, s / alpha, t_piv, alpha]     (2j+2 doubles, device)
// with alpha^2 = beta - c.c and t_piv = (s_piv - c.s) / alpha^2 (Arnoldi;
// QR: t_piv = (s_piv - c.s) / alpha, qr != 0, and the new column's s_new is
// not divided by alpha), and copies g to `gout` (mapped host memory) for
// the host.  The guards themselves stay on the host; when the host declares a
// breakdown the speculative device work is discarded.  c.c and c.s are summed
// in a fixed order, so every rank (same g bits) computes the same
// coefficients.
#include "step.cuh"

namespace {

using namespace kls;

__global__ void __launch_bounds__(kThreads) dcgs2_scalars_kernel(const double* __restrict__ g,
                                                                 int32_t j, int32_t qr,
                                                                 double* __restrict__ coef,
                                                                 double* gout) {
  dcgs2_scalars_block(g, j, qr, coef, gout);
}

}  // namespace

// coef (device, 2j+2) <- the update coefficients of a DCGS2 step from its
// reduced vector g (device, 2j+3); g is also copied to gout (mapped host
// memory, may be NULL).  qr != 0 selects the QR form (ortho.py:369).
KLS_API int kls_dcgs2_scalars(const double* g, int32_t j, int32_t qr, double* coef, double* gout,
                              void* stream) {
  if (g == nullptr || coef == nullptr || j < 0) return fail(KLS_EINVAL, "dcgs2_scalars: bad arguments");
  dcgs2_scalars_kernel<<<1, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(g, j, qr, coef, gout);
  return check_launch("dcgs2_scalars_kernel");
}
