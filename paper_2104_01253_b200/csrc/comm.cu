// Cross-GPU exchange over NVLink peer memory (symmetric buffers).
//
// kls_peer_seg_combine is a reduction's global combine (the paper's
// MPI_Allreduce; ledger site kernels.py:57-59) done as a
// one-shot exchange instead of an NCCL call: every rank copies its exported
// segment-tree nodes (seg.cuh) into its own symmetric buffer, raises an
// epoch flag in every peer's buffer, waits for all peers' flags, then
// evaluates the fixed tree from all ranks' nodes.  Every rank computes the
// same sums in the same order as a one-rank run, so all ranks hold
// bitwise-identical results (the property the replicated host step relies
// on) -- and the result lands directly in page-locked host memory.
// Double-buffered by epoch parity: a rank can only reuse a slot after every
// peer has signalled the following epoch, i.e. after they have finished
// reading it.
//
// kls_peer_signal / kls_stencil7_peer replace the halo exchange: a rank
// signals "my vector for epoch e is written" to its neighbours, and the
// stencil kernel reads the neighbouring x-planes straight from the peers'
// memory once their flags reach e.
//
// Symmetric buffer layout (per rank, identical offsets):
//   uint64 ar_flag[kMaxPeers] | uint64 halo_flag[kMaxPeers] | pad |
//   double slot[2][cap]
// Every spin has a wall-clock timeout (globaltimer) so a missing peer turns
// into an error code instead of a hung GPU.
#include "peer.cuh"
#include "seg.cuh"

#include <cstring>
#include "stencil.cuh"
#include "stencil_tma.cuh"

namespace {

using namespace kls;
using namespace kls::peer;

// A reduction's cross-rank combine: publish this rank's exported tree nodes
// (src, [e][nv]) in its own slot, signal every peer, wait for every peer,
// then every rank evaluates the fixed segment tree from all ranks' exports.
__global__ void __launch_bounds__(kThreads) peer_seg_combine_kernel(const double* __restrict__ src,
                                                                    int nv, double* out, Peers p,
                                                                    uint64_t epoch, int* err) {
  __shared__ int s_ok;
  double* dst = slot(p.buf[p.rank], p.cap, epoch);
  int ids[seg::kMaxExport];
  const int nexp = seg::exports(seg::seg_first(p.rank, p.world),
                                seg::seg_first(p.rank + 1, p.world), ids);
  for (int i = threadIdx.x; i < nexp * nv; i += blockDim.x) dst[i] = src[i];
  seg::Dest d;
  d.out = out;
  d.xstride = nv;
  d.peers = p;
  d.epoch = epoch;
  d.err = err;
  if (!seg::peer_exchange<kThreads, 0>(d, threadIdx.x, &s_ok)) {
    if (threadIdx.x == 0) *err = 1;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) out[i] = __longlong_as_double(0x7ff8000000000000ll);
    return;
  }
  seg::combine_from_slots<kThreads>(d, nv, threadIdx.x, [&](int o, double v) { out[o] = v; });
}

__global__ void peer_signal_kernel(Peers p, int target_mask, uint64_t epoch) {
  const int t = threadIdx.x;
  if (t < p.world && ((target_mask >> t) & 1)) {
    __threadfence_system();
    st_release_sys(halo_flags(p.buf[t]) + p.rank, epoch);
  }
}

// Stencil with peer halos: CTAs whose chunk touches a rank boundary wait for
// the neighbour's flag, then read its plane over NVLink.
__global__ void __launch_bounds__(32 * kSTY) stencil7_peer_kernel(
    const double* __restrict__ x, const double* x_lo, const double* x_hi, double* __restrict__ y,
    int64_t nx, int32_t ny, int32_t nz, int32_t xchunk, const uint64_t* flag_lo,
    const uint64_t* flag_hi, uint64_t epoch, int* err) {
  __shared__ int s_ok;
  __shared__ double tile[kSTY + 2][kSTZ + 2];
  const int64_t xa = static_cast<int64_t>(blockIdx.z) * xchunk;
  const int64_t xb = xa + xchunk < nx ? xa + xchunk : nx;
  const bool need_lo = xa == 0 && x_lo != nullptr;
  const bool need_hi = xb == nx && x_hi != nullptr;
  if (need_lo || need_hi) {
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      bool ok = true;
      if (need_lo) ok = ok && wait_flag(flag_lo, epoch);
      if (need_hi) ok = ok && wait_flag(flag_hi, epoch);
      s_ok = ok;
      if (!ok) *err = 1;
    }
    __syncthreads();
    if (!s_ok) return;
  }
  if (xa >= xb) return;
  stencil7_tile_march(x, x_lo, x_hi, y, nx, ny, nz, xa, xb, tile);
}

int make_peers(Peers& p, void* const* bufs, int rank, int world, int cap) {
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world || bufs == nullptr || cap < 1)
    return fail(KLS_EINVAL, "peer: bad rank/world (%d/%d) or capacity", rank, world);
  for (int r = 0; r < kMaxPeers; ++r) p.buf[r] = r < world ? static_cast<char*>(bufs[r]) : nullptr;
  for (int r = 0; r < world; ++r)
    if (p.buf[r] == nullptr) return fail(KLS_EINVAL, "peer: null buffer for rank %d", r);
  p.rank = rank;
  p.world = world;
  p.cap = cap;
  return KLS_OK;
}

}  // namespace

// ---- peer buffers for callers without a collective allocator --------------
// (C / C++ hosts: one process per GPU, handles exchanged over the caller's
// own bootstrap — MPI, a socket, NCCL's unique-id channel.)

KLS_API size_t kls_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

// Allocate and zero a peer buffer of `bytes` on the current device; writes
// its IPC handle (kls_ipc_handle_bytes() bytes) to `handle`.
KLS_API int kls_peer_buffer_alloc(size_t bytes, void** buf, void* handle) {
  if (buf == nullptr || handle == nullptr || bytes == 0)
    return fail(KLS_EINVAL, "peer_buffer_alloc: bad arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e == cudaSuccess) e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    if (p != nullptr) cudaFree(p);
    return fail(KLS_ECUDA, "peer_buffer_alloc: %s", cudaGetErrorString(e));
  }
  std::memcpy(handle, &h, sizeof(h));
  *buf = p;
  return KLS_OK;
}

// Map another rank's peer buffer (from its handle) into this device.
KLS_API int kls_peer_buffer_open(const void* handle, void** peer_buf) {
  if (handle == nullptr || peer_buf == nullptr) return fail(KLS_EINVAL, "peer_buffer_open: bad arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(peer_buf, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(KLS_ECUDA, "peer_buffer_open: %s", cudaGetErrorString(e));
  return KLS_OK;
}

KLS_API int kls_peer_buffer_close(void* peer_buf) {
  cudaError_t e = cudaIpcCloseMemHandle(peer_buf);
  if (e != cudaSuccess) return fail(KLS_ECUDA, "peer_buffer_close: %s", cudaGetErrorString(e));
  return KLS_OK;
}

KLS_API int kls_peer_buffer_free(void* buf) {
  cudaError_t e = cudaFree(buf);
  if (e != cudaSuccess) return fail(KLS_ECUDA, "peer_buffer_free: %s", cudaGetErrorString(e));
  return KLS_OK;
}

// Bytes of a symmetric peer buffer holding `cap` doubles per slot.
KLS_API size_t kls_peer_buffer_bytes(int32_t cap) {
  return kDataOff + 2 * static_cast<size_t>(cap) * sizeof(double);
}

// Cross-rank combine of a reduction whose world > 1 launch wrote this
// rank's exported tree nodes to `src` ([e][nv], device): every rank
// publishes them in its symmetric buffer and evaluates the fixed segment
// tree into `out` (device or mapped host memory) -- the same bits on every
// rank and as on one GPU.  `epoch` must increase by one per call and be
// identical on all ranks; *err (device int) is set to 1 when a peer does
// not arrive within the timeout.
KLS_API int kls_peer_seg_combine(const double* src, int32_t nv, double* out, void* const* bufs,
                                 int32_t rank, int32_t world, int32_t cap, uint64_t epoch,
                                 int* err, void* stream) {
  Peers p;
  int rc = make_peers(p, bufs, rank, world, cap);
  if (rc) return rc;
  if (nv < 0 || static_cast<int64_t>(nv) * seg::kMaxExport > cap || src == nullptr ||
      out == nullptr || err == nullptr)
    return fail(KLS_EINVAL, "peer_seg_combine: 8 x nv = %d exceeds slot capacity %d",
                8 * nv, cap);
  peer_seg_combine_kernel<<<1, kThreads, 0, static_cast<cudaStream_t>(stream)>>>(src, nv, out, p,
                                                                                  epoch, err);
  return check_launch("peer_seg_combine_kernel");
}

// Raise this rank's halo flag (value epoch) in the buffers of the ranks in
// target_mask, after all prior work on the stream.
KLS_API int kls_peer_signal(void* const* bufs, int32_t rank, int32_t world, int32_t target_mask,
                            uint64_t epoch, void* stream) {
  Peers p;
  int rc = make_peers(p, bufs, rank, world, 1);
  if (rc) return rc;
  peer_signal_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(p, target_mask, epoch);
  return check_launch("peer_signal_kernel");
}

// kls_stencil7 with the neighbouring planes read from peer memory: x_lo /
// x_hi are peer-mapped addresses (or NULL at the physical boundary); the
// kernel first waits until this rank's halo flags from the lower / upper
// neighbour (in its own symmetric buffer `mybuf`) reach `epoch`.
KLS_API int kls_stencil7_peer(const double* x, const double* x_lo, const double* x_hi, double* y,
                              int64_t nx, int64_t ny, int64_t nz, void* mybuf, int32_t rank,
                              uint64_t epoch, int* err, void* stream) {
  if (x == nullptr || y == nullptr || nx < 0 || ny < 0 || nz < 0 || mybuf == nullptr ||
      rank < 0 || rank >= kMaxPeers || err == nullptr)
    return fail(KLS_EINVAL, "stencil7_peer: bad arguments");
  const int64_t plane = ny * nz;
  if (nx * plane == 0) return KLS_OK;
  const uint64_t* flags = reinterpret_cast<const uint64_t*>(static_cast<char*>(mybuf)) + kMaxPeers;
  const uint64_t* flag_lo = rank > 0 ? flags + (rank - 1) : flags;
  const uint64_t* flag_hi = flags + (rank + 1 < kMaxPeers ? rank + 1 : rank);
  const int64_t xchunk = std::min<int64_t>(32, nx);
  dim3 grid;
  if (stencil7_tma_ok(x, ny, nz) && stencil7_grid(nx, ny, nz, xchunk, grid, kTZ, kTY)) {
    CUtensorMap map;
    const int use_map = stencil7_tensor_map(x, nx, ny, nz, &map) ? 1 : 0;
    TmaStencilArgs a{use_map, x, x_lo, x_hi, y, nx, static_cast<int32_t>(ny),
                     static_cast<int32_t>(nz), static_cast<int32_t>(xchunk),
                     x_lo != nullptr ? flag_lo : nullptr, x_hi != nullptr ? flag_hi : nullptr,
                     epoch, err};
    return launch_dependent(stencil7_tma_kernel, grid, dim3(kTThreads), 0,
                            static_cast<cudaStream_t>(stream), "stencil7_tma_kernel", a, map);
  }
  if (ny > INT32_MAX || nz > INT32_MAX || !stencil7_grid(nx, ny, nz, xchunk, grid, kSTZ, kSTY))
    return fail(KLS_EINVAL, "stencil7_peer: grid too large");
  stencil7_peer_kernel<<<grid, dim3(32, kSTY), 0, static_cast<cudaStream_t>(stream)>>>(
      x, x_lo, x_hi, y, nx, static_cast<int32_t>(ny), static_cast<int32_t>(nz),
      static_cast<int32_t>(xchunk), flag_lo, flag_hi, epoch, err);
  return check_launch("stencil7_peer_kernel");
}
