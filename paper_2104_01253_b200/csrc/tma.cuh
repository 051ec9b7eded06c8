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
// used there (the schedule is then the plain round-robin one).
constexpr int64_t kBalanceRounds = 16;

// The schedule as an incremental walk (per chunk: one add and one compare on
// the producer's critical path): round-robin chunks [row, row + R) with row
// stepping by grid * R up to rr_end, then at most one short balanced chunk.
template <int R>
struct ChunkWalk {
  int64_t row, step, rr_end, tail_row, tail_nr;

  // the launch's own CTA (grid = gridDim.x, b = blockIdx.x)
  __device__ __forceinline__ explicit ChunkWalk(int64_t m64)
      : ChunkWalk(m64, gridDim.x, blockIdx.x, kBalanceRounds) {}

  // virtual CTA b of a grid of `grid` (segmented reductions, seg.cuh);
  // with fewer than `balance` whole rounds the remainder is split evenly
  __device__ __forceinline__ ChunkWalk(int64_t m64, int64_t grid, int64_t b, int64_t balance) {
    const int64_t q = m64 / R / grid;  // whole rounds
    step = grid * R;
    row = b * R;
    if (q >= balance) {
      rr_end = m64;  // plain round-robin; the last chunk may be short
      tail_nr = 0;
      tail_row = 0;
    } else {
      rr_end = q * step;
      const int64_t per = ((m64 - rr_end) / 64 + grid - 1) / grid * 64;
      tail_row = rr_end + b * per;
      const int64_t left = m64 - tail_row;
      tail_nr = left < per ? (left > 0 ? left : 0) : per;
    }
  }

  // next chunk: start row r and rows nr (a multiple of 64); false when done
  __device__ __forceinline__ bool next(int64_t& r, int64_t& nr) {
    if (row < rr_end) {
      r = row;
      nr = rr_end - row < R ? rr_end - row : R;
      row += step;
      return true;
    }
    if (tail_nr > 0) {
      r = tail_row;
      nr = tail_nr;
      tail_nr = 0;
      return true;
    }
    return false;
  }
};

}  // namespace tma
}  // namespace kls
