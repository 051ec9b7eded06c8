// Shared helpers for the klsgpu sm_100a kernels.
//
// Layout contract: a basis block Q is column-major with a
// leading dimension `ldq` (rows of storage per column, a multiple of 32
// doubles so every column starts on a 256-byte boundary).  Vectors are plain
// fp64 arrays of `m` rows whose base is 16-byte aligned.  Every kernel
// processes exactly `m` rows (odd tails are handled), never the padding.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include <algorithm>

#include "klsgpu.h"  // status codes; prototypes checked against the definitions

#define KLS_API extern "C" __attribute__((visibility("default")))

namespace kls {

int fail(int code, const char* fmt, ...);
int check_launch(const char* what);
int sm_count();  // SMs of the current device (cached per device)

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Launch `kernel` as the programmatic dependent of the preceding kernel on
// the stream (it may start while that one finishes; it pdl_wait()s before
// touching the predecessor's results).  KLS_PDL=0 launches plainly.
bool pdl_enabled();

template <typename K, typename... Args>
int launch_dependent(K kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     const char* name, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, args...);
  if (e != cudaSuccess) return fail(KLS_ECUDA, "%s launch: %s", name, cudaGetErrorString(e));
  return check_launch(name);
}


}  // namespace kls

// --------------------------------------------------------------------------
// device helpers

// 128-bit load through the read-only (non-coherent) path.  Only for data
// that no thread writes during the kernel.
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ double ld_stream1(const double* p) { return __ldg(p); }

// Load the row pair (r, r+1) of a column; rows >= m read as 0.
template <bool CHECK>
__device__ __forceinline__ double2 load_pair(const double* col, int64_t r, int64_t m) {
  if (!CHECK) return ld_stream2(col + r);
  if (r + 1 < m) return ld_stream2(col + r);
  double2 v = make_double2(0.0, 0.0);
  if (r < m) v.x = ld_stream1(col + r);
  return v;
}

// Same, through the coherent path (for vectors the kernel also writes).
template <bool CHECK>
__device__ __forceinline__ double2 load_pair_rw(const double* col, int64_t r, int64_t m) {
  if (!CHECK) return *reinterpret_cast<const double2*>(col + r);
  if (r + 1 < m) return *reinterpret_cast<const double2*>(col + r);
  double2 v = make_double2(0.0, 0.0);
  if (r < m) v.x = col[r];
  return v;
}

template <bool CHECK>
__device__ __forceinline__ void store_pair(double* col, int64_t r, int64_t m, double2 v) {
  if (!CHECK || r + 1 < m) {
    *reinterpret_cast<double2*>(col + r) = v;
  } else if (r < m) {
    col[r] = v.x;
  }
}

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor finishes; it must pdl_wait() before touching what the
// predecessor writes.  The predecessor pdl_trigger()s once its main work is
// done.  Both are no-ops outside a PDL pair.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reduce-scatter V values across a warp with a butterfly that halves the
// payload at each of the first log2(V) levels, then finishes with a plain
// xor tree.  Costs (V-1) + (5 - log2 V) shuffles instead of 5 V.  On return
// every lane holds the full warp sum of value index `warp_slot<V>(lane)`.
template <int V>
__device__ __forceinline__ double warp_transpose_reduce(double (&v)[V], int lane) {
  static_assert(V == 1 || V == 2 || V == 4 || V == 8 || V == 16, "V power of two <= 16");
  int n = V;
  int o = 16;
#pragma unroll
  for (int lvl = 0; (1 << lvl) < V; ++lvl) {
    const int half = n >> 1;
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < V / 2; ++i) {
      if (i < half) {
        const double keep = upper ? v[i + half] : v[i];
        const double send = upper ? v[i] : v[i + half];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    n = half;
    o >>= 1;
  }
  double r = v[0];
  for (; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// Value index held by `lane` after warp_transpose_reduce<V>.
template <int V>
__device__ __forceinline__ int warp_slot(int lane) {
  int idx = 0;
  int n = V;
  int o = 16;
  while (n > 1) {
    n >>= 1;
    if (lane & o) idx += n;
    o >>= 1;
  }
  return idx;
}
