"""Operators with device-resident data, plus the host-side generators that
build the reference's test problems (reference problems.py).

Operators follow the reference's LinearOperator protocol (problems.py:12-65):
``shape``, ``apply(x)`` (validates, counts ``napply``), ``frobenius_norm()``,
``to_dense()``.  ``apply`` takes a device tensor holding this rank's rows (or
a host array of the global length, which is sliced and uploaded) and returns
a device tensor.  Rows are block-partitioned over the ranks of the active
communicator; ``apply`` exchanges the halo rows a stencil/CSR row needs from
neighbouring ranks before launching the kernel.

Generators (CsrMatrix.from_coo, manteuffel_build, laplace3d, ...) run on the
host with numpy and produce exactly the reference's CSR arrays (same entry
order, same summed values), so device SpMV results are bit-identical.
"""

import io
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, runtime, trace
from .errors import DimensionError, MatrixMarketError

# ---------------------------------------------------------------------------
# device vectors with halo space


class HaloVector:
    """A rank's rows of a vector plus storage for the halo rows an operator
    reads from its neighbours.

    ``local`` is the (aligned) view of the owned rows; ``ext`` is the base the
    CSR column indices address; ``lo``/``hi`` are the halo views (or None).
    """

    def __init__(self, n_local, lo_rows=0, hi_rows=0, contiguous=True):
        dev = runtime.device()
        self.n_local = n_local
        if contiguous:
            # [pad | lo halo | local | hi halo] with local 256-byte aligned
            pad = (-lo_rows) % runtime.ALIGN
            total = pad + lo_rows + n_local + hi_rows
            self.buf = torch.zeros(max(total, 2), dtype=torch.float64, device=dev)
            self.ext_offset = pad
            start = pad + lo_rows
            self.local = self.buf[start : start + n_local]
            self.lo = self.buf[pad : pad + lo_rows] if lo_rows else None
            self.hi = self.buf[start + n_local : start + n_local + hi_rows] if hi_rows else None
        else:
            # [local (padded) | lo plane | hi plane]: halos by separate pointer
            ld = runtime.pad_rows(n_local)
            self.buf = torch.zeros(ld + lo_rows + hi_rows, dtype=torch.float64, device=dev)
            self.ext_offset = 0
            self.local = self.buf[:n_local]
            self.lo = self.buf[ld : ld + lo_rows] if lo_rows else None
            self.hi = self.buf[ld + lo_rows : ld + lo_rows + hi_rows] if hi_rows else None

    @property
    def ext_ptr(self):
        return self.buf.data_ptr() + 8 * self.ext_offset


# ---------------------------------------------------------------------------
# operator protocol


class LinearOperator:
    """Square operator y = A x; subclasses implement ``_launch``.

    ``napply`` counts applications through ``apply`` (one per matvec), which
    the Arnoldi instrumentation asserts against (problems.py:12-33).
    """

    def __init__(self, n, comm=None):
        self.n = int(n)
        self.napply = 0
        self._fro = None
        self.comm = comm if comm is not None else runtime.comm()
        self._scratch = None
        self._partition()

    # -- partition ----------------------------------------------------------
    def _partition(self):
        # rows follow the 24 global reduction segments (64-row units):
        # rank-count-independent reductions, DESIGN.md §6a
        self.segs = self.comm.segs(self.n, runtime.row_unit(self.n))
        self.row_lo, self.row_hi = self.segs.lo, self.segs.hi

    @property
    def m_local(self):
        return self.row_hi - self.row_lo

    @property
    def shape(self):
        return (self.n, self.n)

    # -- vectors ------------------------------------------------------------
    def new_vector(self):
        """A zeroed HaloVector laid out for this operator's kernel."""
        return HaloVector(self.m_local)

    def take(self, x, name="operand"):
        """Validate an operand and return this rank's rows on the device."""
        if isinstance(x, torch.Tensor) and x.is_cuda:
            if x.dim() != 1 or x.numel() != self.m_local:
                raise DimensionError(
                    f"{name} of local length {self.m_local} expected, got {tuple(x.shape)}"
                )
            return x if x.dtype == torch.float64 else x.double()
        if isinstance(x, torch.Tensor):
            # host tensor (pinned for an async copy): this rank's rows only
            if x.dim() != 1 or x.numel() != self.n:
                raise DimensionError(f"{name} of length {self.n} expected, got {tuple(x.shape)}")
            part = x[self.row_lo : self.row_hi].to(torch.float64)
            runtime.XFER["h2d"] += 8 * part.numel()
            return part.to(runtime.device(), non_blocking=part.is_pinned())
        a = np.asarray(x, dtype=np.float64)
        if a.shape != (self.n,):
            raise DimensionError(f"{name} of length {self.n} expected, got {a.shape}")
        return runtime.upload(a[self.row_lo : self.row_hi])

    # -- application ----------------------------------------------------------
    def apply(self, x):
        """y = A x as a new device tensor (counts one application)."""
        xl = self.take(x)
        self.napply += 1
        y = torch.empty(self.m_local, dtype=torch.float64, device=xl.device)
        self.apply_into(xl, y)
        return y

    def apply_into(self, x, y, st=None):
        """Uncounted y = A x on stream ``st`` (default: the current stream).
        ``x`` is a HaloVector (no copy) or a device tensor of the local rows
        (copied into scratch halo storage when the operator needs neighbour
        rows)."""
        if st is None:
            st = runtime.stream_handle()
        if not isinstance(x, (HaloVector, PeerVector)):
            if self._needs_halo():
                if self._scratch is None:
                    self._scratch = self.new_vector()
                self._scratch.local.copy_(x)
                x = self._scratch
            else:
                x = _PlainVector(x)
        self._exchange(x)
        rec = trace._active
        if rec is None:
            self._launch(x, y, st)
        else:
            rec.note("apply", self.apply_bytes())
            with rec.span("apply"):
                self._launch(x, y, st)

    def apply_bytes(self):
        """Algorithmic HBM bytes of one application (x read, y written)."""
        return 16 * self.m_local

    def _needs_halo(self):
        return False

    def _exchange(self, x):
        pass

    def _launch(self, x, y, st):
        raise NotImplementedError

    def op_desc(self):
        """The one-rank apply as plain pointers (include/klsgpu.h KlsOpDesc)
        for the C++ step plan, or None when the operator is not plain."""
        return None

    # -- norms / dense ------------------------------------------------------
    def to_dense(self, max_order=4000):
        if self.n > max_order:
            raise MemoryError(f"dense assembly of order {self.n} refused (limit {max_order})")
        if self.comm.world != 1:
            raise NotImplementedError("to_dense on a row-sharded operator")
        out = np.empty((self.n, self.n), order="F")
        e = torch.zeros(self.n, dtype=torch.float64, device=runtime.device())
        y = torch.empty_like(e)
        for j in range(self.n):
            e[j] = 1.0
            self.apply_into(e, y)
            out[:, j] = y.cpu().numpy()
            e[j] = 0.0
        return out

    def frobenius_norm(self, samples=64, seed=0):
        """Estimated once by probing sampled columns (problems.py:51-65)."""
        if self._fro is None:
            if self.comm.world != 1:
                raise NotImplementedError("probed Frobenius norm on a row-sharded operator")
            t = min(samples, self.n)
            rng = np.random.Generator(np.random.PCG64(seed))
            cols = rng.choice(self.n, size=t, replace=False)
            e = torch.zeros(self.n, dtype=torch.float64, device=runtime.device())
            y = torch.empty_like(e)
            acc = 0.0
            for j in cols:
                e[j] = 1.0
                self.apply_into(e, y)
                acc += float(torch.dot(y, y))
                e[j] = 0.0
            self._fro = float(np.sqrt(acc * self.n / t))
        return self._fro


def _scratch_copy(op, x, peer_ok):
    """A halo-capable copy of a plain local vector for a sharded apply (CGS2
    applies the operator to a basis column, GMRES to its iterate).  With a
    peer link the copy goes into one of TWO peer vectors used alternately:
    before a rank overwrites the buffer of apply k it has passed apply k+1's
    wait on its neighbours' halo flags, which they raise only after their
    apply k -- so no neighbour still reads it.  Otherwise an NCCL halo
    vector."""
    link = runtime.peer_link(op.comm)
    if link is None or not peer_ok:
        if op._scratch is None:
            op._scratch = op._plain_vector()
        op._scratch.local.copy_(x)
        return op._scratch
    pair = op.__dict__.get("_peer_scratch")
    if pair is None:
        pair = op._peer_scratch = [PeerVector(link, op.m_local), PeerVector(link, op.m_local)]
        op._peer_scratch_next = 0
    v = pair[op._peer_scratch_next]
    op._peer_scratch_next ^= 1
    v.local.copy_(x)
    return v


class PeerVector:
    """A vector in NVLink symmetric memory: peers read its rows directly."""

    def __init__(self, link, n_local):
        self.link = link
        self.n_local = n_local
        self.buf, self.peer_ptrs, self._hdl = link.symmetric_vector(runtime.pad_rows(n_local))
        self.local = self.buf[:n_local]
        self.lo = self.hi = None
        self.ext_offset = 0
        self.leased = False

    def release(self):
        """Return the vector to its operator's pool (explicit, same program
        point on every rank)."""
        self.leased = False

    @property
    def ext_ptr(self):
        return self.local.data_ptr()


class _PlainVector:
    """Adapter: a local tensor viewed as a halo-free HaloVector."""

    def __init__(self, t):
        self.local = t
        self.lo = self.hi = None
        self.buf = t
        self.ext_offset = 0

    @property
    def ext_ptr(self):
        return self.local.data_ptr()


def _p2p(ops):
    import torch.distributed as dist

    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def halo_plan(rank, windows):
    """Point-to-point plan of a row-sharded SpMV halo exchange.

    ``windows[q] = (need_lo, own_lo, own_hi, need_hi)``: rank q owns global
    rows [own_lo, own_hi) and its rows read columns [need_lo, need_hi).
    Returns (sends, recvs) for ``rank``: sends are (peer, a, b) slices of the
    local rows; recvs are (peer, "lo"|"hi", a, b) slices of the halo buffers
    (offsets from the start of the lo window [need_lo, own_lo) or the hi
    window [own_hi, need_hi)).
    """
    need_lo, own_lo, own_hi, need_hi = windows[rank]
    sends, recvs = [], []
    for q, (qn_lo, q_lo, q_hi, qn_hi) in enumerate(windows):
        if q == rank:
            continue
        for a, b in ((qn_lo, q_lo), (q_hi, qn_hi)):  # rows of mine that q reads
            x0, x1 = max(a, own_lo), min(b, own_hi)
            if x1 > x0:
                sends.append((q, x0 - own_lo, x1 - own_lo))
        for a, b, side in ((need_lo, own_lo, "lo"), (own_hi, need_hi, "hi")):  # q's rows I read
            x0, x1 = max(a, q_lo), min(b, q_hi)
            if x1 > x0:
                recvs.append((q, side, x0 - a, x1 - a))
    return sends, recvs


class DenseOperator(LinearOperator):
    """Small dense operator (problems.py:68-85), single rank."""


    def __init__(self, a, comm=None):
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise DimensionError(f"square matrix expected, got {a.shape}")
        super().__init__(a.shape[0], comm)
        if self.comm.world != 1:
            raise NotImplementedError("DenseOperator is single-rank")
        self.a = a
        self._dev = runtime.upload(np.ascontiguousarray(a))

    def _launch(self, x, y, st):
        _lib.call("kls_dense_gemv", self._dev.data_ptr(), self.n, self.n, x.local.data_ptr(),
                  y.data_ptr(), st)

    def op_desc(self):
        return _lib.KlsOpDesc(kind=_lib.OP_DENSE, m=self.n, n0=self.n, p0=self._dev.data_ptr())

    def to_dense(self, max_order=None):
        return self.a.copy()

    def frobenius_norm(self, samples=None, seed=None):
        if self._fro is None:
            self._fro = float(np.linalg.norm(self.a))
        return self._fro


class DeviceFunctionOperator(LinearOperator):
    """A user operator given as a device function: ``fn(x)`` maps this rank's
    rows of x (a float64 CUDA tensor) to this rank's rows of A x, with torch
    ops or the caller's own kernels, on the current stream.  The counterpart
    of subclassing the reference's LinearOperator with a numpy ``_matvec``
    (problems.py:12-33): the vector never leaves the GPU.  With more than one
    rank, ``fn`` sees only the local rows and does its own neighbour
    exchange."""

    def __init__(self, n, fn, comm=None):
        super().__init__(n, comm)
        self.fn = fn

    def _launch(self, x, y, st):
        out = self.fn(x.local)
        if not isinstance(out, torch.Tensor) or out.shape != (self.m_local,) or not out.is_cuda:
            raise DimensionError(
                f"operator function must return a CUDA vector of length {self.m_local}")
        y.copy_(out)


# ---------------------------------------------------------------------------
# CSR storage (host) and the device CSR operator


@dataclass
class CsrMatrix:
    """Host CSR with sorted, unique column indices per row (problems.py:88-151).

    A data container: products run on the device through CsrOperator.
    """

    nrows: int
    ncols: int
    indptr: np.ndarray
    indices: np.ndarray
    data: np.ndarray

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals):
        """Build from triplets, summing duplicates in (row, col) order."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        perm = np.lexsort((cols, rows))  # stable: equal keys keep input order
        rows, cols, vals = rows[perm], cols[perm], vals[perm]
        if rows.size:
            first = np.ones(rows.size, dtype=bool)
            first[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
            slot = np.cumsum(first) - 1
            summed = np.zeros(int(slot[-1]) + 1)
            np.add.at(summed, slot, vals)  # sequential in input order
            rows, cols, vals = rows[first], cols[first], summed
        counts = np.bincount(rows, minlength=nrows) if rows.size else np.zeros(nrows, np.int64)
        indptr = np.zeros(nrows + 1, dtype=np.int64)
        np.cumsum(counts, out=indptr[1:])
        return cls(nrows, ncols, indptr, cols, vals)

    @property
    def nnz(self):
        return int(self.indices.size)

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def row_ids(self):
        return np.repeat(np.arange(self.nrows), np.diff(self.indptr))

    def transpose(self):
        return CsrMatrix.from_coo(self.ncols, self.nrows, self.indices, self.row_ids(), self.data)

    def to_dense(self):
        out = np.zeros((self.nrows, self.ncols))
        out[self.row_ids(), self.indices] = self.data
        return out

    def frobenius_norm(self):
        return float(np.linalg.norm(self.data))

    def matvec(self, x):
        """y = A x (problems.py:127-136) computed on the device by
        kls_csr_spmv — bit-identical to the reference's reduceat order — and
        returned as a host array, as the reference returns it."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.ncols,):
            raise DimensionError(f"operand of length {self.ncols} expected, got {x.shape}")
        dev = runtime.device()
        rp = torch.from_numpy(np.ascontiguousarray(self.indptr, dtype=np.int64)).to(dev)
        ci = torch.from_numpy(np.ascontiguousarray(self.indices, dtype=np.int32)).to(dev)
        va = torch.from_numpy(np.ascontiguousarray(self.data, dtype=np.float64)).to(dev)
        xd = torch.zeros(max(self.ncols, 1), dtype=torch.float64, device=dev)
        xd[: self.ncols] = torch.from_numpy(x).to(dev)
        y = torch.empty(max(self.nrows, 1), dtype=torch.float64, device=dev)
        if self.nrows:
            _lib.call("kls_csr_spmv", rp.data_ptr(), ci.data_ptr() if self.nnz else None,
                      va.data_ptr() if self.nnz else None, self.nrows, xd.data_ptr(),
                      y.data_ptr(), runtime.stream_handle())
        return y[: self.nrows].cpu().numpy()


class CsrOperator(LinearOperator):
    """Device-resident CSR operator (problems.py:154-174).

    Each rank uploads its row block; column indices are remapped onto the
    rank's extended vector [lo halo | local | hi halo], where the halo window
    spans the columns its rows touch outside the owned range.
    """

    def __init__(self, csr, comm=None):
        if csr.nrows != csr.ncols:
            raise DimensionError(f"square matrix expected, got {csr.shape}")
        if csr.ncols >= 2**31:
            raise DimensionError("column indices must fit in int32")
        super().__init__(csr.nrows, comm)
        self.csr = csr
        lo, hi = self.row_lo, self.row_hi
        s, e = int(csr.indptr[lo]), int(csr.indptr[hi])
        cols = csr.indices[s:e]
        cmin = int(cols.min()) if cols.size else lo
        cmax = int(cols.max()) if cols.size else hi - 1
        self.halo_lo = max(0, lo - min(cmin, lo))
        self.halo_hi = max(0, max(cmax + 1, hi) - hi)
        base = lo - self.halo_lo  # global row of ext[0] (HaloVector.ext_ptr)
        dev = runtime.device()
        self._set_arrays(torch.from_numpy(csr.indptr[lo : hi + 1] - s).to(dev),
                         torch.from_numpy((cols - base).astype(np.int32)).to(dev),
                         torch.from_numpy(np.ascontiguousarray(csr.data[s:e])).to(dev))

    # rows of at most this many entries are also stored as ELL (coalesced
    # streams, same products and summation order as the CSR kernel)
    ELL_MAX_WIDTH = 8

    def _set_arrays(self, rowptr, col, val):
        self._rowptr, self._col, self._val = rowptr, col, val
        self._rowptr_p = rowptr.data_ptr()
        self._col_p = col.data_ptr()
        self._val_p = val.data_ptr()
        self._plan = None
        self._ell = None
        nrows = rowptr.numel() - 1
        if nrows > 0:
            width = int((rowptr[1:] - rowptr[:-1]).max().item())
            if 1 <= width <= self.ELL_MAX_WIDTH:
                ld = runtime.pad_rows(nrows)
                dev = rowptr.device
                ecol = torch.empty(width * ld, dtype=torch.int32, device=dev)
                evals = torch.empty(width * ld, dtype=torch.float64, device=dev)
                elen = torch.empty(ld, dtype=torch.uint8, device=dev)
                _lib.call("kls_csr_to_ell", self._rowptr_p, self._col_p, self._val_p, nrows, width,
                          ld, ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(),
                          runtime.stream_handle())
                self._ell = (ecol, evals, elen, width, ld)
        self._peer = False
        if self.comm.world > 1:
            self._plan = self._halo_plan()

    @classmethod
    def _device_built(cls, n, band, nnz_fn, build_fn, comm=None):
        """Row block assembled in HBM by a libklsgpu builder.  ``band`` is the
        operator's half bandwidth (halo rows on each side)."""
        if n >= 2**31:
            raise DimensionError("column indices must fit in int32")
        self = cls.__new__(cls)
        LinearOperator.__init__(self, n, comm)
        self.csr = None
        lo, hi = self.row_lo, self.row_hi
        self.halo_lo = min(band, lo)
        self.halo_hi = min(band, n - hi)
        nnz = int(nnz_fn(lo, hi))
        dev = runtime.device()
        rowptr = torch.empty(hi - lo + 1, dtype=torch.int64, device=dev)
        col = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
        build_fn(lo, hi - lo, lo - self.halo_lo, rowptr.data_ptr(), col.data_ptr(), val.data_ptr())
        self._set_arrays(rowptr, col, val)
        return self

    def _needs_halo(self):
        return self.halo_lo > 0 or self.halo_hi > 0

    def _plain_vector(self):
        return HaloVector(self.m_local, self.halo_lo, self.halo_hi, contiguous=True)

    def new_vector(self):
        """Halo-capable vector.  With an NVLink peer link and halos that come
        from the adjacent ranks only, the vector lives in symmetric memory and
        the apply reads the neighbours' rows directly (kls_ell_spmv_peer);
        otherwise the halo window arrives by NCCL send/recv."""
        if not self._peer:
            return self._plain_vector()
        pool = self.__dict__.setdefault("_peer_pool", [])
        for v in pool:
            if not v.leased:
                v.leased = True
                return v
        v = PeerVector(self._link, self.m_local)
        v.leased = True
        pool.append(v)
        return v

    def apply_into(self, x, y, st=None):
        if not isinstance(x, (HaloVector, PeerVector)) and self._needs_halo():
            x = _scratch_copy(self, x, bool(self._peer))
        super().apply_into(x, y, st)

    def _halo_plan(self):
        """Exchange plan from every rank's [need_lo, own_lo, own_hi, need_hi),
        and whether every rank can read its halo from its adjacent ranks'
        vectors over NVLink (decided collectively: all ranks take one path)."""
        c = self.comm
        link = runtime.peer_link(c)
        mine = (self.row_lo - self.halo_lo, self.row_lo, self.row_hi, self.row_hi + self.halo_hi,
                1 if (link is not None and self._ell is not None) else 0)
        import torch.distributed as dist

        allw = [None] * c.world
        dist.all_gather_object(allw, mine, group=c.group)
        wins = [tuple(int(v) for v in w) for w in allw]
        ok = all(w[4] for w in wins)
        for r, (nlo, lo, hi, nhi, _) in enumerate(wins):
            if nlo < lo and (r == 0 or nlo < wins[r - 1][1]):
                ok = False  # lower halo reaches past the adjacent rank
            if nhi > hi and (r == c.world - 1 or nhi > wins[r + 1][2]):
                ok = False
        self._peer = ok
        self._link = link if ok else None
        self._wins = wins
        return halo_plan(c.rank, [w[:4] for w in wins])

    def _exchange(self, x):
        if self._plan is None or isinstance(x, PeerVector):
            return
        import torch.distributed as dist

        sends, recvs = self._plan
        ops = []
        for q, a, b in sends:
            ops.append(dist.P2POp(dist.isend, x.local[a:b], q, group=self.comm.group))
        for q, side, a, b in recvs:
            buf = x.lo if side == "lo" else x.hi
            ops.append(dist.P2POp(dist.irecv, buf[a:b], q, group=self.comm.group))
        _p2p(ops)

    def apply_bytes(self):
        """x and y, plus values (8) and column indices (4) per stored entry,
        and row pointers (8) or ELL row lengths (1) per row."""
        if self._ell is not None:
            return 16 * self.m_local + 12 * self._ell[3] * self.m_local + self.m_local
        return 16 * self.m_local + 12 * int(self._col.numel()) + 8 * (self.m_local + 1)

    def _launch(self, x, y, st):
        if isinstance(x, PeerVector):
            return self._launch_peer(x, y, st)
        if self._ell is not None:
            ecol, evals, elen, width, ld = self._ell
            _lib.call("kls_ell_spmv", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width,
                      self.m_local, ld, x.ext_ptr, y.data_ptr(), st)
            return
        _lib.call("kls_csr_spmv", self._rowptr_p, self._col_p, self._val_p, self.m_local,
                  x.ext_ptr, y.data_ptr(), st)

    def _launch_peer(self, x, y, st):
        """Signal 'my vector is written' to the adjacent ranks, then the ELL
        product reading their rows of the halo window over NVLink."""
        link, r, world = self._link, self.comm.rank, self.comm.world
        mask = (1 << (r - 1) if r > 0 else 0) | (1 << (r + 1) if r + 1 < world else 0)
        x_lo = x_hi = None
        if self.halo_lo > 0:
            lo_prev, hi_prev = self._wins[r - 1][1], self._wins[r - 1][2]
            x_lo = x.peer_ptrs[r - 1] + 8 * (hi_prev - lo_prev - self.halo_lo)
        if self.halo_hi > 0:
            x_hi = x.peer_ptrs[r + 1]
        link.halo_epoch += 1
        rec = trace._active
        if rec is not None and rec.events:
            with rec.span("halo"):
                _lib.call("kls_peer_signal", link.ptrs, r, world, mask, link.halo_epoch, st)
        else:
            _lib.call("kls_peer_signal", link.ptrs, r, world, mask, link.halo_epoch, st)
        ecol, evals, elen, width, ld = self._ell
        b_lo, b_hi = self._halo_rows()
        _lib.call("kls_ell_spmv_peer", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width,
                  self.m_local, ld, x.local.data_ptr(), x_lo, self.halo_lo, x_hi, y.data_ptr(),
                  b_lo, b_hi, link.mybuf, r - 1 if r > 0 else -1, r + 1 if r + 1 < world else -1,
                  link.halo_epoch, link.err_dev, st)

    def _halo_rows(self):
        """(b_lo, b_hi): the leading rows up to the last one with a lower-halo
        column, and the trailing rows from the first one with an upper-halo
        column (window coordinates); the rows between read owned columns only."""
        if getattr(self, "_brows", None) is None:
            col, rp = self._col, self._rowptr
            m, nlo = self.m_local, self.halo_lo
            rows = torch.repeat_interleave(torch.arange(m, device=col.device),
                                           (rp[1:] - rp[:-1]))
            lo_rows = rows[col[: rows.numel()] < nlo]
            hi_rows = rows[col[: rows.numel()] >= nlo + m]
            b_lo = int(lo_rows.max().item()) + 1 if lo_rows.numel() else 0
            b_hi = m - int(hi_rows.min().item()) if hi_rows.numel() else 0
            if b_lo + b_hi > m:  # overlapping boundary bands: all rows wait
                b_lo, b_hi = m, 0
            self._brows = (b_lo, b_hi)
        return self._brows

    def op_desc(self):
        if self.comm.world != 1 or self.m_local == 0:
            return None
        if self._ell is not None:
            ecol, evals, elen, width, ld = self._ell
            return _lib.KlsOpDesc(kind=_lib.OP_ELL, width=width, m=self.m_local, n0=ld,
                                  p0=ecol.data_ptr(), p1=evals.data_ptr(), p2=elen.data_ptr())
        return _lib.KlsOpDesc(kind=_lib.OP_CSR, m=self.m_local, p0=self._rowptr_p,
                              p1=self._col_p, p2=self._val_p)

    def to_dense(self, max_order=4000):
        if self.n > max_order:
            raise MemoryError(f"dense assembly of order {self.n} refused (limit {max_order})")
        if self.csr is None:
            return LinearOperator.to_dense(self, max_order)
        return self.csr.to_dense()

    def frobenius_norm(self, samples=None, seed=None):
        """||data||_F: exact from the host CSR (problems.py:150-151), or summed
        on the device (and over ranks) for a device-built operator."""
        if self._fro is None:
            if self.csr is not None:
                self._fro = self.csr.frobenius_norm()
            else:
                from . import kernels

                if self._ell is not None:
                    # sum over the ELL entry columns (zero-padded, row-major
                    # per column): each a rank-count-independent dot
                    _, evals, _, width, ld = self._ell
                    # the same number of dots on every rank
                    width = self.comm.allreduce_max_int(width)
                    acc = 0.0
                    zero = torch.zeros(max(self.m_local, 2), dtype=torch.float64, device=evals.device)
                    for k in range(width):
                        v = evals[k * ld : k * ld + self.m_local] if k < self._ell[3] else zero[: self.m_local]
                        acc += kernels.dot(v, v, comm=self.comm, segs=self.segs)
                    self._fro = float(np.sqrt(acc))
                else:
                    v = self._val[: int(self._rowptr[-1].item())]
                    if self.comm.world != 1:
                        raise NotImplementedError("Frobenius norm of a sharded CSR without ELL copy")
                    self._fro = float(np.sqrt(kernels.dot(v, v, comm=self.comm) if v.numel() else 0.0))
        return self._fro


# ---------------------------------------------------------------------------
# Manteuffel convection-diffusion (problems.py:177-284)


@dataclass(frozen=True)
class ManteuffelSpec:
    """(1/h^2) M + (beta/2h) N on a k x k grid, m = k^2; defaults L = k+1,
    h = 1."""

    k: int
    beta: float = 0.5
    length: float = None

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k >= 1 required")
        if self.length is None:
            object.__setattr__(self, "length", float(self.k + 1))

    @property
    def h(self):
        return self.length / (self.k + 1)

    @property
    def m(self):
        return self.k * self.k


def _grid5(k):
    """Row/col/kind triplets of the 5-point coupling on a k x k grid in CSR
    order: per row r = blk*k + i, columns r-k, r-1, r, r+1, r+k when inside.
    kind: -1 lower neighbour, 0 diagonal, +1 upper neighbour."""
    r = np.arange(k * k, dtype=np.int64)
    blk, i = np.divmod(r, k)
    parts = [
        (r - k, blk > 0, -1),
        (r - 1, i > 0, -1),
        (r, np.ones_like(i, dtype=bool), 0),
        (r + 1, i < k - 1, 1),
        (r + k, blk < k - 1, 1),
    ]
    cols = np.stack([p[0] for p in parts], axis=1)
    mask = np.stack([p[1] for p in parts], axis=1)
    kind = np.broadcast_to(np.array([p[2] for p in parts]), cols.shape)
    counts = mask.sum(axis=1)
    indptr = np.zeros(k * k + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, cols[mask], kind[mask]


def manteuffel_parts(spec):
    """Unscaled diffusion part M (4 on the diagonal, -1 off) and convection
    part N (-1 below, +1 above), as CSR."""
    k = spec.k
    indptr, cols, kind = _grid5(k)
    mm = CsrMatrix(spec.m, spec.m, indptr, cols.copy(), np.where(kind == 0, 4.0, -1.0))
    off = kind != 0
    rows = np.repeat(np.arange(spec.m), np.diff(indptr))[off]
    n_ptr = np.zeros(spec.m + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=spec.m), out=n_ptr[1:])
    nn = CsrMatrix(spec.m, spec.m, n_ptr, cols[off].copy(), kind[off].astype(np.float64))
    return mm, nn


def manteuffel_build(spec):
    """Assemble A = (1/h^2) M + (beta/2h) N as CSR.

    Same entries and same rounding as the reference's from_coo of the two
    scaled parts: off-diagonals are diff*(-1) + conv*(+-1), the diagonal is
    diff*4 (problems.py:232-245).
    """
    indptr, cols, kind = _grid5(spec.k)
    diff = 1.0 / (spec.h * spec.h)
    conv = spec.beta / (2.0 * spec.h)
    vals = np.where(kind == 0, diff * 4.0, diff * -1.0 + conv * kind.astype(np.float64))
    return CsrMatrix(spec.m, spec.m, indptr, cols.astype(np.int64), vals)


@dataclass(frozen=True)
class EigenvalueTable:
    """Exact spectrum with multiplicities (values sorted ascending)."""

    values: np.ndarray
    unique: np.ndarray
    multiplicity: np.ndarray


def manteuffel_eigenvalues(spec):
    """Closed-form spectrum (problems.py:257-284):
    lambda = (2/h^2) [2 - sqrt(1 - (beta h/2)^2)(cos(l pi/(k+1)) + cos(j pi/(k+1)))]."""
    bh = spec.beta * spec.h
    if abs(bh) > 2.0:
        raise ValueError("beta*h <= 2 required for a real spectrum")
    rad = np.sqrt(1.0 - (bh / 2.0) ** 2)
    th = np.cos(np.arange(1, spec.k + 1) * np.pi / (spec.k + 1))
    values = np.sort(((2.0 / spec.h**2) * (2.0 - rad * (th[:, None] + th[None, :]))).ravel())
    scale = max(abs(values[0]), abs(values[-1]), 1.0)
    unique, mult = [], []
    for v in values:
        if unique and abs(v - unique[-1]) <= 1e-12 * scale:
            mult[-1] += 1
        else:
            unique.append(v)
            mult.append(1)
    return EigenvalueTable(values=values, unique=np.array(unique),
                           multiplicity=np.array(mult, dtype=np.int64))


# ---------------------------------------------------------------------------
# matrix-free 3-D Laplacian (problems.py:287-344)


class StencilLaplace3D(LinearOperator):
    """Matrix-free 7-point Laplacian on an nx x ny x nz Dirichlet grid, x
    slowest.  Ranks own contiguous blocks of x-planes; the neighbouring
    planes arrive by NCCL send/recv before each application."""

    def __init__(self, nx, ny, nz, comm=None):
        if min(nx, ny, nz) < 1:
            raise ValueError("dimensions >= 1 required")
        self.dims = (int(nx), int(ny), int(nz))
        super().__init__(nx * ny * nz, comm)

    def _partition(self):
        # whole x-planes per rank, at the 24 reduction segments' boundaries
        # (unit = one plane, two when the plane has an odd row count)
        nx, ny, nz = self.dims
        self.plane = ny * nz
        self.segs = self.comm.segs(self.n, self.plane)
        self.row_lo, self.row_hi = self.segs.lo, self.segs.hi
        self.x_lo, self.x_hi = self.row_lo // self.plane, self.row_hi // self.plane
        if self.comm.world > 1:
            for r in range(self.comm.world):
                lo, hi = runtime.seg_range(self.n, self.segs.unit, self.comm.world, r)
                if hi <= lo:
                    raise DimensionError(
                        f"laplace3d{self.dims} over {self.comm.world} ranks leaves rank {r} "
                        "without an x-plane")

    def _needs_halo(self):
        return self.comm.world > 1

    def _plain_vector(self):
        lo = self.plane if self.x_lo > 0 else 0
        hi = self.plane if self.x_hi < self.dims[0] else 0
        if self.comm.world == 1:
            lo = hi = 0
        return HaloVector(self.m_local, lo, hi, contiguous=False)

    def new_vector(self):
        """Halo-capable vector.  With an NVLink peer link the vector lives in
        symmetric memory and neighbours read its boundary planes directly
        (kls_stencil7_peer); otherwise halos arrive by NCCL send/recv."""
        link = runtime.peer_link(self.comm) if self.comm.world > 1 else None
        if link is None:
            return self._plain_vector()
        # symmetric allocations need a collective rendezvous (slow): reuse
        # released vectors.  Leases are taken and returned at the same
        # program points on every rank (SPMD), so the pools stay aligned.
        pool = self.__dict__.setdefault("_peer_pool", [])
        for v in pool:
            if not v.leased:
                v.leased = True
                return v
        v = PeerVector(link, self.m_local)
        v.leased = True
        pool.append(v)
        return v

    def apply_into(self, x, y, st=None):
        if not isinstance(x, (HaloVector, PeerVector)) and self._needs_halo():
            x = _scratch_copy(self, x, True)
        super().apply_into(x, y, st)

    def _exchange(self, x):
        if self.comm.world == 1 or isinstance(x, PeerVector):
            return
        rec = trace._active
        if rec is not None and rec.events:
            with rec.span("halo"):
                self._exchange_planes(x)
        else:
            self._exchange_planes(x)

    def _exchange_planes(self, x):
        import torch.distributed as dist

        P, g = self.plane, self.comm.group
        nxl = self.x_hi - self.x_lo
        ops = []
        r = self.comm.rank
        if nxl > 0:
            if self.x_lo > 0:
                ops.append(dist.P2POp(dist.isend, x.local[:P], r - 1, group=g))
                ops.append(dist.P2POp(dist.irecv, x.lo, r - 1, group=g))
            if self.x_hi < self.dims[0]:
                ops.append(dist.P2POp(dist.isend, x.local[(nxl - 1) * P :], r + 1, group=g))
                ops.append(dist.P2POp(dist.irecv, x.hi, r + 1, group=g))
        _p2p(ops)

    def _launch(self, x, y, st):
        _, ny, nz = self.dims
        if isinstance(x, PeerVector):
            return self._launch_peer(x, y, st)
        lo = x.lo.data_ptr() if x.lo is not None else None
        hi = x.hi.data_ptr() if x.hi is not None else None
        _lib.call("kls_stencil7", x.local.data_ptr(), lo, hi, y.data_ptr(),
                  self.x_hi - self.x_lo, ny, nz, st)

    def op_desc(self):
        if self.comm.world != 1 or self.m_local == 0:
            return None
        _, ny, nz = self.dims
        return _lib.KlsOpDesc(kind=_lib.OP_STENCIL7, m=self.m_local, n0=self.x_hi - self.x_lo,
                              n1=ny, n2=nz)

    def _launch_peer(self, x, y, st):
        """Signal 'my vector is written' to the x-neighbours, then run the
        stencil reading their boundary planes over NVLink."""
        link = x.link
        r, world = self.comm.rank, self.comm.world
        nx, ny, nz = self.dims
        lo_ptr = hi_ptr = None
        mask = 0
        if self.x_lo > 0:
            plo, phi = (v // self.plane for v in runtime.seg_range(self.n, self.segs.unit, world, r - 1))
            lo_ptr = x.peer_ptrs[r - 1] + 8 * (phi - plo - 1) * self.plane
            mask |= 1 << (r - 1)
        if self.x_hi < nx:
            hi_ptr = x.peer_ptrs[r + 1]
            mask |= 1 << (r + 1)
        link.halo_epoch += 1
        rec = trace._active
        if rec is not None and rec.events:
            with rec.span("halo"):
                _lib.call("kls_peer_signal", link.ptrs, r, world, mask, link.halo_epoch, st)
        else:
            _lib.call("kls_peer_signal", link.ptrs, r, world, mask, link.halo_epoch, st)
        _lib.call("kls_stencil7_peer", x.local.data_ptr(), lo_ptr, hi_ptr, y.data_ptr(),
                  self.x_hi - self.x_lo, ny, nz, link.mybuf, r, link.halo_epoch, link.err_dev, st)

    def to_csr(self):
        """Host CSR with the same entries (for CSR-path runs and tests)."""
        nx, ny, nz = self.dims
        idx = np.arange(self.n, dtype=np.int64).reshape(self.dims)
        rows = [idx.ravel()]
        cols = [idx.ravel()]
        vals = [np.full(self.n, 6.0)]
        for axis in range(3):
            a = np.take(idx, np.arange(self.dims[axis] - 1), axis=axis).ravel()
            b = np.take(idx, np.arange(1, self.dims[axis]), axis=axis).ravel()
            rows += [a, b]
            cols += [b, a]
            vals += [np.full(a.size, -1.0), np.full(a.size, -1.0)]
        return CsrMatrix.from_coo(self.n, self.n, np.concatenate(rows), np.concatenate(cols),
                                  np.concatenate(vals))

    def frobenius_norm(self, samples=None, seed=None):
        if self._fro is None:
            nx, ny, nz = self.dims
            edges = (nx - 1) * ny * nz + nx * (ny - 1) * nz + nx * ny * (nz - 1)
            self._fro = float(np.sqrt(36.0 * self.n + 2.0 * edges))
        return self._fro


def laplace3d(nx, ny, nz, comm=None):
    return StencilLaplace3D(nx, ny, nz, comm)


def laplace3d_csr_operator(nx, ny, nz, comm=None):
    """The 7-point Laplacian as a CSR operator assembled on the device —
    the same entries as CsrOperator(laplace3d(nx, ny, nz).to_csr()) without
    the host COO assembly."""
    lib = _lib.load()
    st = runtime.stream_handle()

    def nnz(lo, hi):
        return lib.kls_lap7_nnz(nx, ny, nz, lo, hi)

    def build(lo, nrows, base, rp, cp, vp):
        _lib.call("kls_build_lap7_csr", nx, ny, nz, lo, nrows, base, rp, cp, vp, st)

    return CsrOperator._device_built(nx * ny * nz, ny * nz, nnz, build, comm)


def manteuffel_operator(spec, comm=None):
    """CsrOperator(manteuffel_build(spec)) assembled on the device (same
    entries and rounding; diff and conv computed on the host as the
    reference does, problems.py:235-236)."""
    lib = _lib.load()
    st = runtime.stream_handle()
    k = spec.k
    diff = 1.0 / (spec.h * spec.h)
    conv = spec.beta / (2.0 * spec.h)

    def nnz(lo, hi):
        return lib.kls_mant5_nnz(k, lo, hi)

    def build(lo, nrows, base, rp, cp, vp):
        _lib.call("kls_build_mant5_csr", k, lo, nrows, base, diff, conv, rp, cp, vp, st)

    return CsrOperator._device_built(k * k, k, nnz, build, comm)


def band_random_operator(m, band=1000, per_row=7, seed=2525, comm=None):
    """Config 5's Arnoldi operator (SURVEY.md §8d's alternative: a random
    banded operator whose halos stay with the adjacent ranks): order m,
    per_row entries per row spread over the band |i - j| <= band, hashed
    columns and values in [-1, 1), assembled on the device
    (kls_build_band_csr; host restatement oracle.band_random_coo, bitwise
    equal through kls.CsrMatrix.from_coo)."""
    if per_row > min(m, 2 * band + 1):
        raise ValueError("per_row must be <= min(m, 2 band + 1)")
    st = runtime.stream_handle()

    def nnz(lo, hi):
        return (hi - lo) * per_row

    def build(lo, nrows, base, rp, cp, vp):
        _lib.call("kls_build_band_csr", m, band, per_row, seed, lo, nrows, base, rp, cp, vp, st)

    return CsrOperator._device_built(m, band, nnz, build, comm)


# ---------------------------------------------------------------------------
# Matrix Market coordinate format (problems.py:364-489)


_MM_SYMMETRY_SIGN = {"general": None, "symmetric": 1.0, "skew-symmetric": -1.0}


def _mm_text(source):
    """The whole Matrix Market text of a path, an open file or the text itself."""
    if hasattr(source, "read"):
        return source.read()
    if isinstance(source, str) and source.lstrip().startswith("%%MatrixMarket"):
        return source
    with open(source, "r", encoding="ascii") as f:
        return f.read()


def parse_matrix_market(source):
    """Real/integer coordinate Matrix Market -> CsrMatrix (general, symmetric,
    skew-symmetric) -- the reference's reader contract (problems.py:368-469:
    accepted headers, symmetric expansion, MatrixMarketError with the 1-based
    line of the first offending line).  One tokenising pass over the text,
    then whole-array parsing and checks; only an error is located line by
    line."""
    text = _mm_text(source)
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    head = lines[0].split() if lines else []
    if len(head) != 5 or head[0] != "%%MatrixMarket":
        raise MatrixMarketError("not a Matrix Market header", line=1)
    obj, fmt, field, sym = (t.lower() for t in head[1:])
    if (obj, fmt) != ("matrix", "coordinate"):
        raise MatrixMarketError(f"only 'matrix coordinate' files are read, not {obj} {fmt}", line=1)
    if field not in ("real", "integer"):
        raise MatrixMarketError(f"field {field!r} is not real", line=1)
    if sym not in _MM_SYMMETRY_SIGN:
        raise MatrixMarketError(f"symmetry {sym!r} is not supported", line=1)
    # significant lines (not blank, not comments) with their line numbers
    body = [(n + 1, t.split()) for n, raw in enumerate(lines[1:], start=1)
            for t in (raw.strip(),) if t and not t.startswith("%")]
    if not body:
        raise MatrixMarketError("no size line", line=len(lines))
    size_ln, size_tok = body[0]
    if len(size_tok) != 3:
        raise MatrixMarketError("the size line must read 'rows cols nnz'", line=size_ln)
    try:
        nr, nc, nnz = (int(v) for v in size_tok)
    except ValueError:
        raise MatrixMarketError("size entries must be integers", line=size_ln) from None
    if min(nr, nc, nnz) < 0:
        raise MatrixMarketError("size entries must be non-negative", line=size_ln)
    entries = body[1:]
    n = len(entries)
    ln = np.array([e[0] for e in entries], dtype=np.int64)
    width_ok = np.array([len(e[1]) == 3 for e in entries], dtype=bool)
    tok = np.array([e[1] if len(e[1]) == 3 else ("1", "1", "0") for e in entries],
                   dtype=object).reshape(-1, 3)
    parse_ok = np.ones(n, dtype=bool)
    try:
        ij = tok[:, :2].astype(np.int64)
        v = tok[:, 2].astype(np.float64)
    except (ValueError, OverflowError):  # rare: find the unparsable lines
        ij = np.ones((n, 2), dtype=np.int64)
        v = np.zeros(n)
        for t, (a_, b_, c_) in enumerate(tok):
            try:
                ij[t] = (int(a_), int(b_))
                v[t] = float(c_)
            except ValueError:
                parse_ok[t] = False
                ij[t], v[t] = (1, 1), 0.0
    in_bounds = (ij[:, 0] >= 1) & (ij[:, 0] <= nr) & (ij[:, 1] >= 1) & (ij[:, 1] <= nc)
    skew_ok = (ij[:, 0] != ij[:, 1]) | (v == 0.0) if sym == "skew-symmetric" else np.ones(n, bool)
    # per line, the reference's check order: count, shape, parse, bounds, skew
    fails = [(np.arange(n) >= nnz, lambda t: f"entries beyond the declared {nnz}"),
             (~width_ok, lambda t: "an entry line must read 'row col value'"),
             (~parse_ok, lambda t: "unparsable entry"),
             (~in_bounds, lambda t: f"entry ({ij[t, 0]}, {ij[t, 1]}) outside the {nr}x{nc} matrix"),
             (~skew_ok, lambda t: "skew-symmetric matrices have a zero diagonal")]
    any_bad = np.zeros(n, dtype=bool)
    for mask, _ in fails:
        any_bad |= mask
    if np.any(any_bad):
        t = int(np.argmax(any_bad))
        msg = next(m for mask, m in fails if mask[t])
        raise MatrixMarketError(msg(t), line=int(ln[t]))
    if n != nnz:
        raise MatrixMarketError(f"{n} entries for {nnz} declared", line=len(lines))
    rows, cols = ij[:, 0] - 1, ij[:, 1] - 1
    sign = _MM_SYMMETRY_SIGN[sym]
    if sign is not None:  # mirror the off-diagonal entries
        off = rows != cols
        rows, cols, v = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                         np.concatenate([v, sign * v[off]]))
    return CsrMatrix.from_coo(nr, nc, rows, cols, v)


def write_matrix_market(csr, target, symmetry="general", comment=None):
    """Coordinate real general text of the stored entries (values as Python
    float reprs, so a re-read is exact)."""
    if symmetry != "general":
        raise ValueError("only general output is supported")
    out = ["%%MatrixMarket matrix coordinate real general"]
    out += [f"% {c}" for c in (comment.splitlines() if comment else [])]
    out.append(f"{csr.nrows} {csr.ncols} {csr.nnz}")
    out += [f"{i} {j} {float(x)!r}" for i, j, x in
            zip((csr.row_ids() + 1).tolist(), (np.asarray(csr.indices) + 1).tolist(), csr.data)]
    text = "\n".join(out) + "\n"
    if hasattr(target, "write"):
        target.write(text)
    else:
        with open(target, "w", encoding="ascii") as f:
            f.write(text)
