// Device-side scalar step of DCGS2, shared by the standalone kernel
// (step.cu, kls_dcgs2_scalars) and the Gram kernels' last CTA (gram.cuh,
// kls_gram_dcgs2_step): from g = [c(0:j), beta, s(0:j), s_piv, aw.aw] it
// writes coef = [c, s / alpha (QR: s), t_piv, alpha] and copies g to gout.
// Called by every thread of one CTA (any multiple of 32 threads up to 1024).
#pragma once

#include "common.cuh"

namespace kls {

__device__ __forceinline__ void dcgs2_scalars_block(const double* g, int j, int qr, double* coef,
                                                    double* gout) {
  __shared__ double red[2][32];
  __shared__ double s_alpha;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  double cc = 0.0, cs = 0.0;
  for (int i = tid; i < j; i += blockDim.x) {
    const double c = g[i];
    cc = fma(c, c, cc);
    cs = fma(c, g[j + 1 + i], cs);
  }
  cc = warp_sum(cc);
  cs = warp_sum(cs);
  if (lane == 0) {
    red[0][warp] = cc;
    red[1][warp] = cs;
  }
  __syncthreads();
  if (tid == 0) {
    double scc = 0.0, scs = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      scc += red[0][w];
      scs += red[1][w];
    }
    const double beta = g[j];
    const double s_piv = g[2 * j + 1];
    const double alpha_sq = beta - scc;
    const double alpha = sqrt(alpha_sq > 0.0 ? alpha_sq : 2.2250738585072014e-308);
    coef[2 * j] = qr ? (s_piv - scs) / alpha : (s_piv - scs) / (alpha * alpha);
    coef[2 * j + 1] = alpha;
    s_alpha = alpha;
  }
  __syncthreads();
  const double alpha = s_alpha;
  for (int i = tid; i < j; i += blockDim.x) {
    coef[i] = g[i];
    coef[j + i] = qr ? g[j + 1 + i] : g[j + 1 + i] / alpha;
  }
  if (gout != nullptr)
    for (int i = tid; i < 2 * j + 3; i += blockDim.x) gout[i] = g[i];
}

}  // namespace kls
