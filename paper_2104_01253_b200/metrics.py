"""Stability metrics on run artifacts (reference metrics.py:41-104).

Evaluation helpers, not part of the instrumented path: they never touch a
ledger.  Device tensors are evaluated by the library's own kernels (the
Gram and fused update + norm kernels, streamed a column or two at a time,
O(m) extra memory, reduced over the rank-count-independent tree); host
arrays with numpy.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import runtime
from .errors import DimensionError
from .problems import LinearOperator

DEFAULT_STRIDE = 5


@dataclass(frozen=True)
class StabilityReport:
    scheme: str
    step: int
    loo: float
    rre: float
    n_forward_converged: int = -1
    invariant_dim: int = -1
    kappa: float = float("nan")

    def __post_init__(self):
        if self.loo < 0.0 or self.rre < 0.0:
            raise ValueError("metrics are non-negative")
        if self.n_forward_converged > max(self.step, self.invariant_dim):
            raise ValueError("converged count cannot exceed the step index")


def _is_dev(x):
    return isinstance(x, torch.Tensor) and x.is_cuda


def _layout(comm, segs):
    comm = comm or runtime.comm()
    if comm.world > 1 and segs is None:
        raise DimensionError("a row-sharded metric needs the rows' layout (segs=, e.g. op.segs)")
    return comm, segs


def loss_of_orthogonality(Q, comm=None, segs=None):
    """||I - Q^T Q||_F.  A device Q streams through the library's Gram
    kernel two columns at a time (kls_mv_trans_mv: Q^T [q_c, q_c+1]), with
    the rank-count-independent reduction -- no k x k cuBLAS product and no
    extra device memory."""
    if _is_dev(Q):
        from . import kernels

        comm, segs = _layout(comm, segs)
        k = Q.shape[1]
        g = np.zeros((k, k))
        for c in range(0, k, 2):
            cols = Q[:, c : min(c + 2, k)]
            g[:, c : c + cols.shape[1]] = kernels.mv_trans_mv(Q, cols, comm=comm, segs=segs)
        return float(np.linalg.norm(np.eye(k) - g))
    Q = np.asarray(Q, dtype=np.float64)
    return float(np.linalg.norm(np.eye(Q.shape[1]) - Q.T @ Q))


def _col_residual_sq(y, Q, coef, comm, segs):
    """||y - Q coef||^2 over all ranks, y overwritten (the fused-norm update,
    kls_mv_times_mat_add_mv with nrm_out)."""
    from . import _lib, kernels

    k = len(coef)
    ws, wsb = runtime.workspace(max(k, 1))
    st = runtime.stream_handle()
    B = kernels._aligned_block(Q[:, :k]) if k else None
    bp, ldb, _, m = kernels._cols(B, "Q") if k else (None, 2, 0, y.numel())
    yd = y.contiguous()
    c = np.ascontiguousarray(coef, dtype=np.float64)

    def launch(o, sp):
        _lib.call("kls_mv_times_mat_add_mv_host", yd.data_ptr(), max(m + (m & 1), 2), m, 1, bp,
                  ldb, k, c.ctypes.data if k else None, -1.0, 1.0, o.data_ptr(), sp, ws, wsb, st)

    return float(kernels._reduce(comm, segs, 1, launch)[0].item())


def representation_error_qr(A, Q, R, comm=None, segs=None):
    """||A - Q R||_F / ||A||_F.  Device Q: column by column through the
    fused update + norm kernel (O(m) extra memory)."""
    if _is_dev(Q):
        from . import kernels

        comm, segs = _layout(comm, segs)
        R = np.asarray(R, dtype=np.float64)
        num = den = 0.0
        for j in range(R.shape[1]):
            a = A[:, j] if _is_dev(A) else runtime.as_device_vector(np.asarray(A)[:, j], Q.shape[0])
            a = a.to(torch.float64).clone()
            den += kernels.dot(a, a, comm=comm, segs=segs)
            num += _col_residual_sq(a, Q, R[: Q.shape[1], j], comm, segs)
        return 0.0 if den == 0.0 else float(np.sqrt(num / den))
    A = np.asarray(A, dtype=np.float64)
    denom = np.linalg.norm(A)
    if denom == 0.0:
        return 0.0
    return float(np.linalg.norm(A - np.asarray(Q) @ np.asarray(R)) / denom)


def representation_error_arnoldi(op, Q, H, comm=None, segs=None):
    """||A Q_k - Q_{k+1} H||_F / ||A||_F for k+1 basis columns and a
    (k+1)-by-k extended H (metrics.py:72-92).  Device Q: streamed one column
    at a time (A q_j, then the fused update + norm with H[:, j]) -- O(m)
    memory, so it runs at config 3's size where A Q would not fit."""
    H = np.asarray(H, dtype=np.float64)
    k = H.shape[1]
    if Q.shape[1] != k + 1 or H.shape[0] != k + 1:
        raise DimensionError(
            f"expected basis k+1 columns and (k+1)-by-k H, got {tuple(Q.shape)} and {H.shape}")
    if k == 0:
        return 0.0
    denom = op.frobenius_norm() if isinstance(op, LinearOperator) else float(np.linalg.norm(op))
    if denom == 0.0:
        return 0.0
    if _is_dev(Q):
        comm = comm or getattr(op, "comm", None)
        segs = segs if segs is not None else getattr(op, "segs", None)
        comm, segs = _layout(comm, segs)
        num = 0.0
        y = torch.empty(Q.shape[0], dtype=torch.float64, device=Q.device)
        for j in range(k):
            op.apply_into(Q[:, j].contiguous(), y)
            nz = int(np.max(np.nonzero(H[:, j])[0])) + 1 if np.any(H[:, j]) else 0
            num += _col_residual_sq(y, Q, H[:nz, j], comm, segs)
        return float(np.sqrt(num)) / denom
    Q = np.asarray(Q, dtype=np.float64)
    a = np.asarray(op, dtype=np.float64)
    return float(np.linalg.norm(a @ Q[:, :k] - Q @ H) / denom)


def forward_error_count(computed, table, tol):
    from .eig import match_eigenvalues

    return match_eigenvalues(computed, table, tol).n_matched
