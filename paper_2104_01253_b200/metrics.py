"""Stability metrics on run artifacts (reference metrics.py:41-104).

Evaluation helpers, not part of the instrumented path: they never touch a
ledger.  Device tensors are evaluated on the device (cuBLAS through torch,
summed over ranks), host arrays with numpy.
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


def _sum_ranks(t, comm=None):
    comm = comm or runtime.comm()
    return comm.allreduce_(t)


def loss_of_orthogonality(Q, comm=None):
    """||I - Q^T Q||_F."""
    if _is_dev(Q):
        g = _sum_ranks(Q.T @ Q, comm)
        return float(torch.linalg.norm(torch.eye(g.shape[0], dtype=g.dtype, device=g.device) - g))
    Q = np.asarray(Q, dtype=np.float64)
    return float(np.linalg.norm(np.eye(Q.shape[1]) - Q.T @ Q))


def representation_error_qr(A, Q, R, comm=None):
    """||A - Q R||_F / ||A||_F."""
    if _is_dev(Q):
        A = A if _is_dev(A) else runtime.upload(np.asarray(A))
        Rt = torch.as_tensor(np.asarray(R), dtype=torch.float64, device=Q.device)
        num = _sum_ranks(torch.sum((A - Q @ Rt) ** 2).reshape(1), comm)
        den = _sum_ranks(torch.sum(A * A).reshape(1), comm)
        return 0.0 if float(den) == 0.0 else float(torch.sqrt(num / den))
    A = np.asarray(A, dtype=np.float64)
    denom = np.linalg.norm(A)
    if denom == 0.0:
        return 0.0
    return float(np.linalg.norm(A - np.asarray(Q) @ np.asarray(R)) / denom)


def representation_error_arnoldi(op, Q, H, comm=None):
    """||A Q_k - Q_{k+1} H||_F / ||A||_F for k+1 basis columns and a
    (k+1)-by-k extended H (metrics.py:72-92)."""
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
        AQ = torch.stack([op.apply(Q[:, j].contiguous()) for j in range(k)], dim=1)
        Ht = torch.as_tensor(H, device=Q.device)
        num = _sum_ranks(torch.sum((AQ - Q @ Ht) ** 2).reshape(1), comm)
        return float(torch.sqrt(num)) / denom
    Q = np.asarray(Q, dtype=np.float64)
    a = np.asarray(op, dtype=np.float64)
    return float(np.linalg.norm(a @ Q[:, :k] - Q @ H) / denom)


def forward_error_count(computed, table, tol):
    from .eig import match_eigenvalues

    return match_eigenvalues(computed, table, tol).n_matched
