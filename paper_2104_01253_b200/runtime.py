"""Device plumbing: device/stream selection, the row partition over ranks,
reduction workspaces, pinned staging buffers.

PyTorch is used for device memory, streams and torch.distributed (NCCL)
only; all arithmetic on the path runs in libklsgpu.so.

Row partition: every distributed object (operator, vector,
basis block) is split into contiguous row blocks, one per rank, in rank
order — the paper's SPMD model.  A single process is the
world-size-1 case of the same code.  The blocks follow the 24 global
segments of the rank-count-independent reductions (csrc/seg.cuh, DESIGN.md
§6a): rank r of N owns segments [24 r / N, 24 (r + 1) / N), so every
reduction gives the same bits on 1, 2, 3, 4, 6 or 8 GPUs.
"""

import ctypes


import numpy as np
import torch

from . import _lib

ALIGN = 32  # doubles: 256-byte column alignment for Q

# host<->device bytes moved by the package (bench.py's e2e accounting)
XFER = {"h2d": 0, "d2h": 0}


def pad_rows(m):
    """Leading dimension for an m-row column block."""
    return max(ALIGN, (m + ALIGN - 1) // ALIGN * ALIGN)


_cuda_ok = None


def device():
    global _cuda_ok
    if not _cuda_ok:
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_2104_01253_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists"
            )
        _cuda_ok = True
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle():
    return torch.cuda.current_stream().cuda_stream


def ptr(t):
    """Device address of a tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


# ---------------------------------------------------------------------------
# communicator


class Comm:
    """Ranks of torch.distributed (NCCL) or the single-process world."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        if dist.is_available() and dist.is_initialized():
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        self.allreduce_calls = 0

    def backend(self):
        import torch.distributed as dist

        return dist.get_backend(self.group) if self.world > 1 else "none"

    def barrier(self):
        import torch.distributed as dist

        if self.world > 1:
            dist.barrier(group=self.group)

    def shares_devices(self):
        """True when two ranks of this comm drive the same GPU."""
        if self.world == 1:
            return False
        if getattr(self, "_shares", None) is None:
            import socket

            import torch.distributed as dist

            me = (socket.gethostname(), torch.cuda.current_device())
            got = [None] * self.world
            dist.all_gather_object(got, me, group=self.group)
            self._shares = len(set(got)) < self.world
        return self._shares

    def allreduce_max_int(self, v):
        """Max of a host integer over the ranks."""
        if self.world == 1:
            return int(v)
        import torch.distributed as dist

        dev = "cpu" if self.backend() == "gloo" else device()
        t = torch.tensor([int(v)], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())

    def allreduce_max_float(self, v):
        """Max of a host float over the ranks."""
        if self.world == 1:
            return float(v)
        import torch.distributed as dist

        dev = "cpu" if self.backend() == "gloo" else device()
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return float(t.item())

    def segs(self, m, unit=None):
        """The reduction layout of an m-row object split over this comm
        (unit: row_unit(m) by default, a stencil passes its x-plane)."""
        return Segs(m, row_unit(m) if unit is None else unit, self.world, self.rank)


    def combine_(self, blocks, count):
        """NCCL path of a reduction's cross-rank combine: `blocks` (device,
        >= 8 * count) holds this rank's exported tree nodes ([e][count]);
        returns the global values (device, count) — the same bits as the
        peer path and as one rank."""
        import torch.distributed as dist

        mine = blocks[: SEG_MAX_EXPORT * count].contiguous()
        if self.backend() == "gloo":  # host all_gather, then back to the device
            parts = [torch.empty(SEG_MAX_EXPORT * count, dtype=torch.float64)
                     for _ in range(self.world)]
            dist.all_gather(parts, mine.cpu(), group=self.group)
            g = torch.stack(parts).to(blocks.device)
        else:
            g = torch.zeros((self.world, SEG_MAX_EXPORT * count), dtype=torch.float64,
                            device=blocks.device)
            dist.all_gather_into_tensor(g, mine, group=self.group)
        out = torch.empty(count, dtype=torch.float64, device=blocks.device)
        _lib.call("kls_seg_combine", g.data_ptr(), count, count, self.world, out.data_ptr(),
                  stream_handle())
        self.allreduce_calls += 1
        return out

    def allreduce_(self, t):
        """In-place sum over ranks (the one global reduction of a step)."""
        if self.world > 1:
            import torch.distributed as dist

            if self.backend() == "gloo" and t.is_cuda:
                h = t.cpu()
                dist.all_reduce(h, group=self.group)
                t.copy_(h)
            else:
                dist.all_reduce(t, group=self.group)
            self.allreduce_calls += 1
        return t

    def allreduce_host(self, arr):
        """Sum a small host array over ranks (returns a new numpy array)."""
        arr = np.asarray(arr, dtype=np.float64)
        if self.world == 1:
            return arr.copy()
        t = torch.from_numpy(arr.copy()).to(device())
        self.allreduce_(t)
        return t.cpu().numpy()


def row_unit(m):
    """Partition unit of an m-row object: 64 rows, or fewer for small m so
    that every one of the 24 segments gets rows (no rank without rows for
    N <= 24); even, and a function of m only (rank-count independent)."""
    return max(2, min(64, 2 * (m // 48)))


def block_range(n, parts, index):
    base, extra = divmod(n, parts)
    lo = index * base + min(index, extra)
    return lo, lo + base + (1 if index < extra else 0)


# ---------------------------------------------------------------------------
# the rank-count-independent segment tree (csrc/seg.cuh; the same arithmetic)

SEG_G = 24
SEG_NODES = 39
SEG_ROOT = 38
SEG_MAX_EXPORT = 8


def seg_row(m, unit, k):
    """Global row where segment k (0..24) starts."""
    units = -(-m // unit)
    return min(m, unit * (units * k // SEG_G))


def seg_first(rank, world):
    return rank * SEG_G // world


def seg_range(m, unit, world, rank):
    """Rank's global rows [lo, hi): segments [24 r / N, 24 (r + 1) / N)."""
    return seg_row(m, unit, seg_first(rank, world)), seg_row(m, unit, seg_first(rank + 1, world))


def _node_lo(n):
    return n if n < 24 else 3 * (n - 24) if n < 32 else 6 * (n - 32) if n < 36 else \
        12 * (n - 36) if n < 38 else 0


def _node_hi(n):
    return n + 1 if n < 24 else 3 * (n - 24) + 3 if n < 32 else 6 * (n - 32) + 6 if n < 36 else \
        12 * (n - 36) + 12 if n < 38 else 24


def _node_parent(n):
    return 24 + n // 3 if n < 24 else 32 + (n - 24) // 2 if n < 32 else \
        36 + (n - 32) // 2 if n < 36 else 38 if n < 38 else -1


def _node_children(n):
    if n < 24:
        return ()
    if n < 32:
        return (3 * (n - 24), 3 * (n - 24) + 1, 3 * (n - 24) + 2)
    if n < 36:
        return (24 + 2 * (n - 32), 25 + 2 * (n - 32))
    if n < 38:
        return (32 + 2 * (n - 36), 33 + 2 * (n - 36))
    return (36, 37)


def seg_exports(rank, world):
    """The tree nodes a rank exports (maximal complete subtrees of its
    segments), left to right."""
    a, b = seg_first(rank, world), seg_first(rank + 1, world)
    ids, pos = [], a
    while pos < b:
        node = pos
        while True:
            p = _node_parent(node)
            if p < 0 or _node_lo(p) != pos or not (a <= _node_lo(p) and _node_hi(p) <= b):
                break
            node = p
        ids.append(node)
        pos = _node_hi(node)
    return ids


def _fold(n, val):
    c = _node_children(n)
    if len(c) == 3:
        return (val[c[0]] + val[c[1]]) + val[c[2]]
    return val[c[0]] + val[c[1]]


def seg_local_nodes(segvals, rank, world):
    """Host restatement of a rank's local tree: segvals (nseg x count) ->
    its exported node values (nexp x count), numpy float64 adds in the
    kernels' order (test scaffolding and reference for the device)."""
    a, b = seg_first(rank, world), seg_first(rank + 1, world)
    val = {}
    for leaf in range(a, b):
        val[leaf] = np.asarray(segvals[leaf - a], dtype=np.float64)
    for n in range(SEG_G, SEG_NODES):
        if a <= _node_lo(n) and _node_hi(n) <= b:
            val[n] = _fold(n, val)
    return np.array([val[i] for i in seg_exports(rank, world)])


def seg_combine_host(blocks, world):
    """Host restatement of kls_seg_combine: blocks[r] = rank r's exported
    node values (nexp_r x count) -> the root (count)."""
    val = {}
    for r in range(world):
        for e, nid in enumerate(seg_exports(r, world)):
            val[nid] = np.asarray(blocks[r][e], dtype=np.float64)
    for n in range(SEG_G, SEG_NODES):
        if n not in val and all(c in val for c in _node_children(n)):
            val[n] = _fold(n, val)
    return val[SEG_ROOT]


class Segs:
    """KlsSegs of one row space (an operator's or a QR block's rows): the
    global row count, the partition unit, and this rank's place."""

    def __init__(self, m, unit, world, rank):
        if unit % 2:
            unit *= 2  # segments start 16-byte aligned
        self.m, self.unit, self.world, self.rank = int(m), int(unit), int(world), int(rank)
        self.lo, self.hi = seg_range(self.m, self.unit, self.world, self.rank)
        self.nexp = len(seg_exports(self.rank, self.world))
        self.c = _lib.KlsSegs(self.m, self.unit, self.world, self.rank)
        self.ptr = ctypes.addressof(self.c)

    @property
    def m_local(self):
        return self.hi - self.lo


_default_comm = None


def comm():
    """The communicator operators bind to when none is given."""
    global _default_comm
    import torch.distributed as dist

    live = dist.is_available() and dist.is_initialized()
    if _default_comm is None or (live and _default_comm.world == 1 and dist.get_world_size() > 1):
        _default_comm = Comm()
    return _default_comm


def set_comm(c):
    global _default_comm
    _default_comm = c


# ---------------------------------------------------------------------------
# workspaces and staging


class Workspace:
    """Zeroed reduction workspace for one stream (tickets reset themselves).

    Grows on demand; a replaced buffer is kept alive (``_old``) because work
    already queued on the stream may still use it.  Callers must not cache
    the pointer across calls that could grow it.
    """

    def __init__(self):
        self._buf = None
        self._bytes = 0
        self._old = []
        self._need = {}

    def get(self, kmax, m=0):
        kmax = int(max(kmax, 8))
        key = (kmax, int(m))
        need = self._need.get(key)
        if need is None:
            need = self._need[key] = int(_lib.load().kls_workspace_bytes(int(m), kmax))
        if self._buf is None or need > self._bytes:
            if self._buf is not None:
                self._old.append(self._buf)
            self._buf = torch.zeros(need, dtype=torch.uint8, device=device())
            self._bytes = need
        return self._buf.data_ptr(), self._bytes


_workspaces = {}


def workspace(kmax):
    return workspace_for(stream_handle(), kmax)


def workspace_for(stream, kmax, m=0):
    """(pointer, bytes) of the reduction workspace of `stream` for reductions
    over m local rows with up to kmax basis columns.  Replaced buffers stay
    alive, so a returned pointer remains valid."""
    key = (torch.cuda.current_device(), stream)
    ws = _workspaces.get(key)
    if ws is None:
        ws = _workspaces[key] = Workspace()
    return ws.get(kmax, m)


class Staging:
    """Pinned host buffer pair for the per-step scalar round trip."""

    def __init__(self, n):
        self.n = 0
        self._grow(max(n, 64))

    def _grow(self, n):
        self.n = n
        self.host_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
        self.host_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
        self.dev_out = torch.empty(n, dtype=torch.float64, device=device())
        self.dev_in = torch.empty(n, dtype=torch.float64, device=device())

    def ensure(self, n):
        if n > self.n:
            self._grow(max(n, 2 * self.n))

    def fetch(self, count):
        """D2H of dev_out[:count]; blocks until it lands; returns a numpy copy
        (the pinned buffer is reused by the next fetch)."""
        h = self.host_out[:count]
        XFER["d2h"] += 8 * count
        h.copy_(self.dev_out[:count], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return h.numpy().copy()

    def push(self, values):
        """H2D of a small host vector into dev_in (ordered on the stream).

        Safe to reuse the pinned buffer: every step synchronizes the stream in
        fetch() before the next push overwrites host_in.
        """
        values = np.asarray(values, dtype=np.float64)
        count = values.size
        self.ensure(count)
        self.host_in[:count].numpy()[:] = values
        XFER["h2d"] += 8 * count
        self.dev_in[:count].copy_(self.host_in[:count], non_blocking=True)
        return self.dev_in[:count]


def upload(arr):
    """Blocking host->device copy of a small array (non-hot paths)."""
    XFER["h2d"] += 8 * int(np.size(arr))
    return torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64)).to(device())


def as_device_vector(x, n_local, lo=0, name="vector"):
    """Accept a numpy array of the global length (sliced to this rank) or a
    device tensor of the local length; return a fresh float64 device vector."""
    if isinstance(x, torch.Tensor):
        if x.dim() != 1:
            raise ValueError(f"{name} must be 1-D")
        if x.numel() == n_local:
            return x.to(device=device(), dtype=torch.float64).clone()
        x = x.detach().cpu().numpy()
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 1:
        raise ValueError(f"{name} must be 1-D")
    if a.size != n_local:
        a = a[lo : lo + n_local]
    return torch.from_numpy(np.ascontiguousarray(a)).to(device())


# ---------------------------------------------------------------------------
# NVLink peer link (symmetric memory)


class _CudaView:
    """__cuda_array_interface__ of raw device memory (torch.as_tensor wraps
    it without a copy)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


class _IpcBuffer:
    """A peer buffer allocated through the C-ABI (kls_peer_buffer_alloc,
    zeroed cudaMalloc) and mapped into every rank by CUDA IPC handles
    exchanged over the process group: works when ranks share a GPU (where
    symmetric memory refuses) and for any host without a collective
    allocator.  Collective."""

    def __init__(self, comm, nbytes):
        import torch.distributed as dist

        lib = _lib.load()
        hbytes = int(lib.kls_ipc_handle_bytes())
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * hbytes)()
        _lib.call("kls_peer_buffer_alloc", nbytes, ctypes.byref(own), handle)
        handles = [None] * comm.world
        dist.all_gather_object(handles, bytes(handle), group=comm.group)
        self.own = own.value
        self.opened = []
        ptrs = []
        for r, h in enumerate(handles):
            if r == comm.rank:
                ptrs.append(self.own)
                continue
            p = ctypes.c_void_p()
            hb = (ctypes.c_char * hbytes).from_buffer_copy(h)
            _lib.call("kls_peer_buffer_open", hb, ctypes.byref(p))
            self.opened.append(p.value)
            ptrs.append(p.value)
        self.ptrs = ptrs
        self.tensor = torch.as_tensor(_CudaView(self.own, nbytes), device=device())

    def __del__(self):
        try:
            for p in self.opened:
                _lib.call("kls_peer_buffer_close", p)
            _lib.call("kls_peer_buffer_free", self.own)
        except Exception:  # interpreter shutdown
            pass


class PeerLink:
    """Peer buffers of one process group, mapped into every peer GPU.

    Carries the one-shot combine of every reduction (the per-step Gram
    scalars among them) and the halo flags of peer-read operators
    (csrc/comm.cu).  Two allocators: torch symmetric memory (one rank per
    GPU), or CUDA-IPC buffers from the C-ABI (kls_peer_buffer_alloc / open;
    used when ranks share a GPU, or with KLS_PEER=ipc).  Allocation and
    rendezvous are collective: every rank must create the link / vectors in
    the same order (they do: the solvers are SPMD).
    """

    CAP = 8192  # doubles per exchange slot (8 exported nodes x count <= CAP)

    def __init__(self, comm, mode="symm"):
        import torch.distributed as dist

        self.comm = comm
        self.mode = mode
        self.rank, self.world = comm.rank, comm.world
        if self.world > 8:
            raise RuntimeError("peer link supports up to 8 ranks (one NVLink domain)")
        group = comm.group if comm.group is not None else dist.group.WORLD
        self._group_name = group.group_name
        nbytes = int(_lib.load().kls_peer_buffer_bytes(self.CAP))
        if mode == "ipc":
            self._ipc = _IpcBuffer(comm, nbytes)
            self.buf = self._ipc.tensor
            ptrs = self._ipc.ptrs
        else:
            import torch.distributed._symmetric_memory as symm_mem

            self.buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device())
            self.buf.zero_()
            self.hdl = symm_mem.rendezvous(self.buf, self._group_name)
            ptrs = [int(p) for p in self.hdl.buffer_ptrs]
        self.ptrs = (ctypes.c_void_p * self.world)(*ptrs)
        self.mybuf = int(ptrs[self.rank])
        self.err_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        from ._engine import _mapped

        self.err_dev = _mapped(self.err_host.data_ptr())
        self.ar_epoch = 0
        self.halo_epoch = 0
        torch.cuda.synchronize()
        comm.barrier()

    def symmetric_vector(self, n):
        """A zeroed device vector mapped into every peer plus every rank's
        pointer to its copy.  Collective; ranks may ask for different
        lengths (uneven row blocks): every copy gets the largest."""
        nmax = self.comm.allreduce_max_int(max(n, 2))
        if self.mode == "ipc":
            b = _IpcBuffer(self.comm, 8 * nmax)
            return b.tensor.view(torch.float64), list(b.ptrs), b
        import torch.distributed._symmetric_memory as symm_mem

        t = symm_mem.empty(nmax, dtype=torch.float64, device=device())
        t.zero_()
        hdl = symm_mem.rendezvous(t, self._group_name)
        return t, [int(p) for p in hdl.buffer_ptrs], hdl

    def take_epochs(self, n):
        """Reserve n consecutive exchange epochs; returns the first."""
        first = self.ar_epoch + 1
        self.ar_epoch += n
        return first

    def seg_combine(self, src_ptr, count, out_ptr, stream):
        """Cross-rank combine of a reduction's exported tree nodes (src,
        [e][count]) into out: the fixed segment tree, same bits everywhere."""
        if count * SEG_MAX_EXPORT > self.CAP:
            raise RuntimeError(f"peer combine of {count} values exceeds the slot ({self.CAP})")
        self.ar_epoch += 1
        _lib.call("kls_peer_seg_combine", src_ptr, count, out_ptr, self.ptrs, self.rank,
                  self.world, self.CAP, self.ar_epoch, self.err_dev, stream)
        self.comm.allreduce_calls += 1

    def check(self):
        if int(self.err_host[0]) != 0:
            raise RuntimeError("NVLink peer exchange timed out (a rank did not arrive)")


def peer_link(comm):
    """The comm's PeerLink, or None (single rank, disabled by KLS_PEER=0, or
    no peer mapping possible, in which case NCCL carries the traffic).
    Ranks sharing a GPU (or KLS_PEER=ipc) use CUDA-IPC buffers."""
    import os

    env = os.environ.get("KLS_PEER", "1")
    if comm.world == 1 or env == "0":
        return None
    if getattr(comm, "_peer", None) is None and not getattr(comm, "_peer_failed", False):
        mode = "ipc" if (env == "ipc" or comm.shares_devices()) else "symm"
        try:
            comm._peer = PeerLink(comm, mode)
        except Exception as exc:  # transport selection only; compute is unchanged
            if comm.backend() != "nccl":
                raise
            import warnings

            warnings.warn(f"NVLink peer link unavailable ({exc}); using NCCL collectives")
            comm._peer_failed = True
            comm._peer = None
    return getattr(comm, "_peer", None)


def init_distributed():
    """One process per rank from torchrun's environment (RANK, LOCAL_RANK,
    WORLD_SIZE, MASTER_*): the GPU is LOCAL_RANK % device count; NCCL when
    every rank has its own GPU, gloo (bootstrap and host values only -- the
    data path goes over CUDA-IPC peer buffers) when ranks share one.
    Returns the default Comm (world 1 without torchrun)."""
    import os

    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local % ndev)
    if world > 1 and not dist.is_initialized():
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        if local_world > ndev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local % ndev))
    return comm()


def shutdown_distributed():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        c = comm()
        c.barrier()
        dist.destroy_process_group()
