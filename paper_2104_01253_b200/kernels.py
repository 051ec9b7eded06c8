"""Instrumented device kernels (reference kernels.py:1-84).

Same contract as the reference: these are the only operations that
synchronize across ranks, each call records its kernel class and nominal
flops (global m) in the ledger, and ``mv_trans_mv`` is exactly one
reduction (one allreduce) regardless of its width, including an empty
basis block.  Operands are device tensors holding this rank's rows; a basis
block B is an (m_local, k) view with unit row stride (column-major, as the
expansions store it).  Reduced values come back to the host as numpy.
"""

import numpy as np
import torch

from . import _lib, runtime
from . import ledger as _ledger
from .errors import DimensionError


def _aligned_block(B):
    """B itself when it is a column-major view the kernels accept (16-byte
    aligned columns, even leading dimension), else a padded copy."""
    m, k = B.shape
    ok = B.stride(0) == 1 and (k <= 1 or B.stride(1) >= m)
    if ok:
        ld = B.stride(1) if k > 1 else max(m + (m & 1), 2)
        ok = B.data_ptr() % 16 == 0 and (k <= 1 or ld % 2 == 0)
    if ok:
        return B
    buf = torch.zeros((max(k, 1), runtime.pad_rows(m)), dtype=torch.float64, device=B.device)
    buf[:k, :m].copy_(B.T)
    return buf[:k, :m].T


def _cols(B, name):
    """(pointer, ld, k) of a column-major (m, k) device view."""
    if not isinstance(B, torch.Tensor) or not B.is_cuda:
        raise DimensionError(f"{name} must be a CUDA tensor")
    if B.dim() == 1:
        B = B[:, None]
    if B.dim() != 2:
        raise DimensionError(f"{name} must be 2-D, got shape {tuple(B.shape)}")
    m, k = B.shape
    if k == 0:
        return 0, max(m, 2), 0, m
    if B.stride(0) != 1 or (k > 1 and B.stride(1) < m):
        raise DimensionError(f"{name} must be column-major with unit row stride")
    ld = B.stride(1) if k > 1 else max(m + (m & 1), 2)
    return B.data_ptr(), ld, k, m


def _global_m(m_local, comm):
    if comm.world == 1:
        return m_local
    t = torch.tensor([float(m_local)], dtype=torch.float64, device=runtime.device())
    comm.allreduce_(t)
    return int(t.item())


def _reduce(comm, segs, count, launch):
    """Run a reducing kernel and combine it over the ranks: launch(out,
    segs_ptr) writes into the device tensor `out` the result (one rank) or
    this rank's exported tree nodes (a (8, count) block); the combine follows
    the fixed segment tree, so the value does not depend on the number of
    ranks (csrc/seg.cuh)."""
    dev = runtime.device()
    if comm.world == 1:
        out = torch.zeros(max(count, 1), dtype=torch.float64, device=dev)
        launch(out, segs.ptr if segs is not None else None)
        return out[:count]
    if segs is None:
        raise DimensionError("a row-sharded reduction needs the rows' layout (segs=, e.g. op.segs)")
    blocks = torch.zeros((runtime.SEG_MAX_EXPORT, max(count, 1)), dtype=torch.float64, device=dev)
    launch(blocks, segs.ptr)
    flat = blocks.view(-1)
    link = runtime.peer_link(comm)
    if link is not None:
        out = torch.empty(max(count, 1), dtype=torch.float64, device=dev)
        link.seg_combine(flat.data_ptr(), count, out.data_ptr(), runtime.stream_handle())
        torch.cuda.current_stream().synchronize()
        link.check()
        return out[:count]
    return comm.combine_(flat, count)


def dot(x, y, ledger=None, comm=None, m_global=None, segs=None):
    """x . y over all ranks; one reduction (MvDot)."""
    comm = comm or runtime.comm()
    if x.shape != y.shape or x.dim() != 1:
        raise DimensionError(f"dot needs equal-length vectors, got {tuple(x.shape)} and {tuple(y.shape)}")
    ws, wsb = runtime.workspace(1)
    st = runtime.stream_handle()
    out = _reduce(comm, segs, 1, lambda o, sp: _lib.call(
        "kls_mv_trans_mv", None, 2, x.numel(), 0, x.data_ptr(), y.data_ptr(), None, 1, 0,
        o.data_ptr(), sp, ws, wsb, st))
    if ledger is not None:
        m = m_global if m_global is not None else _global_m(x.numel(), comm)
        ledger.record(_ledger.MV_DOT, flops=2 * m)
    return float(out[0].item())


def norm2(x, ledger=None, comm=None, m_global=None, segs=None):
    """Euclidean norm via one dot reduction."""
    return float(np.sqrt(dot(x, x, ledger=ledger, comm=comm, m_global=m_global, segs=segs)))


def mv_trans_mv(B, X, ledger=None, comm=None, m_global=None, segs=None):
    """B^T X over all ranks (k x l numpy result); exactly one reduction.

    X may have any number of columns; they are processed two at a time into
    one output block, combined over the ranks once.
    """
    comm = comm or runtime.comm()
    if isinstance(B, torch.Tensor) and B.dim() == 2 and B.is_cuda:
        B = _aligned_block(B)
    bp, ldb, k, m = _cols(B, "B")
    Xv = X[:, None] if X.dim() == 1 else X
    if Xv.shape[0] != m:
        raise DimensionError(f"row mismatch: B is {tuple(B.shape)}, X is {tuple(X.shape)}")
    l = Xv.shape[1]
    ws, wsb = runtime.workspace(k)
    st = runtime.stream_handle()
    n = k * l

    def launch(o, sp):
        # columns c, c+1 -> outputs [c k, (c + 2) k); with several ranks each
        # launch's exported nodes (stride nx k) land in the same columns of
        # the (8, n) export block
        for c in range(0, l, 2):
            nx = min(2, l - c)
            if k == 0:
                continue
            x0 = Xv[:, c].clone()  # fresh, aligned allocations
            x1 = Xv[:, c + 1].clone() if nx == 2 else None
            x1p = None if x1 is None else x1.data_ptr()
            if o.dim() == 1:
                _lib.call("kls_mv_trans_mv", bp, ldb, m, k, None, x0.data_ptr(), x1p, nx, 0,
                          o[c * k :].data_ptr(), sp, ws, wsb, st)
            else:
                tmp = torch.zeros((runtime.SEG_MAX_EXPORT, nx * k), dtype=torch.float64,
                                  device=o.device)
                _lib.call("kls_mv_trans_mv", bp, ldb, m, k, None, x0.data_ptr(), x1p, nx, 0,
                          tmp.data_ptr(), sp, ws, wsb, st)
                o[:, c * k : c * k + nx * k].copy_(tmp)

    out = _reduce(comm, segs, n, launch)
    if ledger is not None:
        mg = m_global if m_global is not None else _global_m(m, comm)
        ledger.record(_ledger.MV_TRANS_MV, flops=2 * mg * k * l)
    return out[:n].cpu().numpy().reshape((l, k)).T.copy()


def mv_times_mat_add_mv(Y, B, S, sign=1.0, scale=1.0, ledger=None, comm=None, m_global=None):
    """Y <- scale*Y + sign*B@S in place (zero reductions); returns Y."""
    comm = comm or runtime.comm()
    if isinstance(B, torch.Tensor) and B.dim() == 2 and B.is_cuda:
        B = _aligned_block(B)
    bp, ldb, k, m = _cols(B, "B")
    Yv = Y[:, None] if Y.dim() == 1 else Y
    Yw = _aligned_block(Yv) if Yv.is_cuda else Yv
    S = np.asarray(S, dtype=np.float64)
    if S.ndim == 1:
        S = S[:, None]
    l = Yv.shape[1]
    if S.shape != (k, l) or Yv.shape[0] != m:
        raise DimensionError(
            f"nonconformal update: Y {tuple(Y.shape)}, B {tuple(B.shape)}, S {S.shape}")
    if ledger is not None:
        mg = m_global if m_global is not None else _global_m(m, comm)
        ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * mg * k * l)
    Sd = runtime.upload(S.T.ravel()) if k else None  # column-major k x l
    st = runtime.stream_handle()
    for c in range(0, l, 2):
        lc = min(2, l - c)
        yp, ldy, _, _ = _cols(Yw[:, c : c + lc], "Y")
        sp = Sd[c * k :].data_ptr() if k else None
        _lib.call("kls_mv_times_mat_add_mv", yp, ldy, m, lc, bp if k else None, ldb, k, sp,
                  float(sign), float(scale), None, None, None, 0, st)
    if Yw is not Yv:
        Yv.copy_(Yw)
    return Y
