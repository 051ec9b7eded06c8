// mbarrier + bulk-async-copy (TMA engine, cp.async.bulk) helpers for the
// shared-memory-staged streaming kernels.  SASS: SYNCS.* and UBLKCP.
#pragma once

#include <stdint.h>

namespace kls {
namespace tma {

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "KLS_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KLS_WAIT_%=;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}


// Chunk schedule of the persistent streaming kernels over the first m64
// rows (m64 a multiple of 64), chunk size R.  Chunks are dealt round-robin
// (chunk k * grid + b to CTA b — neighbouring CTAs stream neighbouring
// chunks, the pattern HBM serves best).  When there are only a few whole
// rounds (m up to ~2e6 rows on 148 SMs), the rows left after the last whole
// round are instead split into grid equal pieces (multiples of 64 rows, one
// short chunk per CTA) rather than dealt as whole chunks to some CTAs while
// the others idle: at m = 1e6 (977 chunks) K1 / K2 at j = 50 take 73 / 65 us
// instead of 77 / 72.  At many rounds the split gains nothing, so it is not
// used there (the schedule is then the plain round-robin one).  Returns
// false past the CTA's last chunk; nr is a multiple of 64.
constexpr int64_t kBalanceRounds = 16;

// q: sched_rounds<R>(m64), computed once per kernel (a 64-bit division)
template <int R>
__device__ __forceinline__ int64_t sched_rounds(int64_t m64) {
  return m64 / R / gridDim.x;
}

template <int R>
__device__ __forceinline__ bool sched_chunk(int64_t it, int64_t q, int64_t m64, int64_t& row,
                                            int64_t& nr) {
  const int64_t grid = gridDim.x, b = blockIdx.x;
  if (q >= kBalanceRounds) {
    const int64_t c = it * grid + b;
    row = c * R;
    if (row >= m64) return false;
    nr = m64 - row < R ? m64 - row : R;
    return true;
  }
  if (it < q) {
    row = (it * grid + b) * R;
    nr = R;
    return true;
  }
  if (it > q) return false;
  const int64_t base = q * grid * R;
  const int64_t per = ((m64 - base) / 64 + grid - 1) / grid * 64;
  row = base + b * per;
  nr = m64 - row < per ? m64 - row : per;
  return nr > 0;
}

}  // namespace tma
}  // namespace kls
