// NVLink peer-memory primitives shared by the one-shot collectives
// (comm.cu) and the Gram kernels with a fused allreduce epilogue (gram.cuh).
#pragma once

#include <stdint.h>

namespace kls {
namespace peer {

constexpr int kMaxPeers = 8;
constexpr size_t kDataOff = 256;
constexpr uint64_t kTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct Peers {
  char* buf[kMaxPeers];  // symmetric buffer base of every rank (peer-mapped)
  int rank;
  int world;
  int cap;  // doubles per slot
};

__device__ __forceinline__ uint64_t* ar_flags(char* b) { return reinterpret_cast<uint64_t*>(b); }
__device__ __forceinline__ uint64_t* halo_flags(char* b) {
  return reinterpret_cast<uint64_t*>(b) + kMaxPeers;
}
__device__ __forceinline__ double* slot(char* b, int cap, uint64_t epoch) {
  return reinterpret_cast<double*>(b + kDataOff) + (epoch & 1) * static_cast<size_t>(cap);
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// spin until *flag >= epoch; false on timeout
__device__ __forceinline__ bool wait_flag(const uint64_t* flag, uint64_t epoch) {
  if (ld_acquire_sys(flag) >= epoch) return true;
  const uint64_t t0 = now_ns();
  while (ld_acquire_sys(flag) < epoch) {
    if (now_ns() - t0 > kTimeoutNs) return false;
    __nanosleep(64);
  }
  return true;
}

}  // namespace peer
}  // namespace kls
