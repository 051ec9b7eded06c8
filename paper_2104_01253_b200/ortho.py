"""Left-looking QR push states on the device (reference ortho.py).

``dcgs2`` (Dcgs2State, ortho.py:326-413): one fused reduction per pushed
column; the pending column is reorthogonalized, normalized (Pythagorean
norm) and emitted during the next push, fused into one pass over Q by
kls_dcgs2_update in its QR form (w' = a - Q s_full, no 1/alpha);
``finalize`` flushes the last column with a CGS2 pass (two reductions).
``cgs2`` (Cgs2State, ortho.py:139-158): three reductions per column.

Q lives on the device; R and the scalar bookkeeping on the host.
"""

import os

import numpy as np
import torch

from . import ledger as _ledger
from . import runtime
from ._engine import Engine
from .errors import BreakdownError, DimensionError, UnknownSchemeError
from .ledger import SyncLedger

_EPS = np.finfo(np.float64).eps

SCHEME_IDS = ("cgs2", "dcgs2")
DELAYED_SCHEMES = ("dcgs2",)


class _RowSpace:
    """Minimal operator stand-in that fixes the row partition of a QR run."""

    def __init__(self, m, comm=None):
        self.comm = comm if comm is not None else runtime.comm()
        self.segs = self.comm.segs(m, runtime.row_unit(m))
        self.row_lo, self.row_hi = self.segs.lo, self.segs.hi
        self.shape = (m, m)

    @property
    def m_local(self):
        return self.row_hi - self.row_lo


class QrState:
    """Shared device storage and bookkeeping (ortho.py:39-117)."""

    scheme_id = None

    def __init__(self, m, n_cap, ledger=None, comm=None):
        self.m = m
        self.n_cap = n_cap
        self.ledger = ledger if ledger is not None else SyncLedger()
        self.space = _RowSpace(m, comm)
        self.eng = Engine(self.space, max(n_cap, 1))
        self._r = np.zeros((n_cap, n_cap))
        self.ncols = 0
        self.npushed = 0
        self.last_coeffs = None
        self.last_alpha = None
        e = self.eng
        self._a = torch.zeros(e.ld, dtype=torch.float64, device=e.vbuf.device)[: e.ml]

    @property
    def q(self):
        return self.eng.block(self.ncols)

    @property
    def r(self):
        return self._r[: self.npushed, : self.npushed]

    def _take(self, a, readonly=False):
        """Column a on the device: a CUDA float64 column is used in place when
        the caller only reads it (readonly), else copied into scratch."""
        e = self.eng
        if isinstance(a, torch.Tensor) and a.is_cuda:
            if a.dim() != 1 or a.numel() != e.ml:
                raise DimensionError(f"column of local length {e.ml} expected, got {tuple(a.shape)}")
            if self.npushed >= self.n_cap:
                raise DimensionError("state capacity exhausted")
            if (readonly and a.dtype == torch.float64 and a.is_contiguous()
                    and a.data_ptr() % 16 == 0 and a.device == e.vbuf.device):
                return a  # read in place: the kernels never write the pushed column
            self._a.copy_(a)
        else:
            a = np.asarray(a, dtype=np.float64)
            if a.shape != (self.m,):
                raise DimensionError(f"column of length {self.m} expected, got {a.shape}")
            self._a.copy_(torch.from_numpy(a[self.space.row_lo : self.space.row_hi]))
        if self.npushed >= self.n_cap:
            raise DimensionError("state capacity exhausted")
        return self._a

    def _check_finite(self, nrm2):
        if not np.isfinite(nrm2):
            raise ValueError("non-finite column")

    def _emit_host(self, coeffs, alpha):
        j = self.ncols
        self._r[: len(coeffs), j] = coeffs
        self._r[j, j] = alpha
        self.last_coeffs = np.asarray(coeffs, dtype=np.float64)
        self.last_alpha = alpha
        self.ncols += 1

    def adopt(self, qcol):
        """Append an externally orthonormalized column (no reductions)."""
        if self.npushed != self.ncols:
            raise DimensionError("cannot adopt while a column is pending")
        self.eng.col(self.ncols).copy_(self._take_any(qcol))
        self._r[self.ncols, self.ncols] = 1.0
        self.ncols += 1
        self.npushed += 1

    def _take_any(self, x):
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x
        x = np.asarray(x, dtype=np.float64)
        return runtime.upload(x[self.space.row_lo : self.space.row_hi] if x.size == self.m else x)

    def adopt_block(self, V):
        for k in range(V.shape[1]):
            self.adopt(V[:, k])

    def push(self, a):
        raise NotImplementedError

    def finalize(self):
        """Flush pending work; returns (Q device view, R host copy)."""
        return self.q, self.r.copy()

    def _guard_alpha(self, alpha, scale):
        if not alpha > _EPS * np.sqrt(self.m) * scale:
            raise BreakdownError(
                f"column {self.npushed} is dependent at working precision "
                f"(norm {alpha:.3e} against scale {scale:.3e})",
                kind="dependent", column=self.npushed)


class Cgs2State(QrState):
    """CGS with full reorthogonalization: 3 reductions per column."""

    scheme_id = "cgs2"

    def push(self, a):
        e = self.eng
        m = self.m
        v = self._take(a)
        j = self.ncols
        r = e.project(j, v, xnorm=True)
        s, scale2 = r[:j].copy(), float(r[j])
        self._check_finite(scale2)
        scale = float(np.sqrt(scale2))
        self.ledger.record(_ledger.MV_TRANS_MV, flops=2 * m * j)
        c = e.subtract_and_project(v, j, s)  # one pass over Q for both
        self.ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * j)
        self.ledger.record(_ledger.MV_TRANS_MV, flops=2 * m * j)
        nrm2 = e.subtract_projection(v, j, c, want_norm=True)
        self.ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * j)
        self.ledger.record(_ledger.MV_DOT, flops=2 * m)
        alpha = float(np.sqrt(nrm2))
        self.last_coeffs, self.last_alpha = s + c, alpha
        self._guard_alpha(alpha, scale)
        self.npushed += 1
        e.divide_into(e.col(j), v, alpha)
        self._emit_host(s + c, alpha)


class Dcgs2State(QrState):
    """Delayed CGS2: one fused reduction per column (ortho.py:326-413)."""

    scheme_id = "dcgs2"

    def __init__(self, m, n_cap, ledger=None, comm=None):
        super().__init__(m, n_cap, ledger, comm)
        e = self.eng
        self._w = torch.zeros(e.ld, dtype=torch.float64, device=e.vbuf.device)[: e.ml]
        self._s = None  # first-projection coefficients of the pending column
        self._wscale = 0.0
        self._pending = False
        # the update is queued with device-computed coefficients before the
        # host has checked the step (as _DelayedArnoldi._step_ahead); w' goes
        # to a spare buffer so a breakdown leaves the pending column intact
        self._lookahead = os.environ.get("KLS_LOOKAHEAD", "1") != "0"
        self._w2 = (torch.zeros(e.ld, dtype=torch.float64, device=e.vbuf.device)[: e.ml]
                    if self._lookahead else None)
        self._slot = 0

    def push(self, a):
        e = self.eng
        m = self.m
        x = self._take(a, readonly=True)
        if not self._pending:
            nrm2 = e.sqnorm(x)  # local norm of the column, not counted
            self._check_finite(nrm2)
            self._w.copy_(x)
            self._s = np.zeros(0)
            self._wscale = float(np.sqrt(nrm2))
            self._pending = True
            self.npushed += 1
            return
        j = self.ncols
        # [Q, w]^T [w, a] plus a.a (the next pending column's local scale)
        if self._lookahead:
            slot = self._slot
            self._slot = 1 - slot
            e.gram_ahead(j, self._w, x, slot, qr=True)
            e.update_ahead(j, self._w, self._w2, x, divide=False)
            g = e.wait_slot(slot, 2 * j + 3)
        else:
            g = e.gram_dcgs2(j, self._w, x)
        self._check_finite(g[2 * j + 2])
        self.ledger.record(_ledger.MV_TRANS_MV, flops=2 * m * (j + 1) * 2)
        c = g[:j].copy()
        beta = float(g[j])
        s_new = g[j + 1 : 2 * j + 1].copy()
        s_piv = float(g[2 * j + 1])
        # finish the pending column (ortho.py:378-399)
        if not np.sqrt(max(beta, 0.0)) > _EPS * np.sqrt(m) * self._wscale:
            raise BreakdownError(f"column {j} is dependent at working precision",
                                 kind="dependent", column=j)
        alpha_sq = beta - float(c @ c)
        self.ledger.add_flops(2 * j)
        if not alpha_sq > beta * _EPS * _EPS:
            raise BreakdownError(f"cancellation in the delayed norm of column {j}",
                                 kind="pythagorean", column=j)
        alpha = float(np.sqrt(alpha_sq))
        self.ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * j)
        # lagged coefficient against the just-emitted q (ortho.py:369)
        s_piv = (s_piv - float(c @ s_new)) / alpha
        self.ledger.add_flops(2 * j)
        s_full = np.append(s_new, s_piv)
        self.ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * (j + 1))
        # one pass: Q(:, j) = (w - Q c)/alpha ; w = a - Q s_new - q_j s_piv
        if self._lookahead:  # already queued; adopt its w'
            self._w, self._w2 = self._w2, self._w
        else:
            e.dcgs2_update(j, self._w, x, c, s_full, alpha, divide=False)
        self._emit_host(self._s + c, alpha)
        self._s = s_full
        self._wscale = float(np.sqrt(g[2 * j + 2]))
        self.npushed += 1

    def finalize(self):
        if self._pending:
            e = self.eng
            m = self.m
            j = self.ncols
            c = e.project(j, self._w, xnorm=False) if j else np.zeros(0)
            self.ledger.record(_ledger.MV_TRANS_MV, flops=2 * m * j)
            nrm2 = e.subtract_projection(self._w, j, c, want_norm=True)
            self.ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * j)
            self.ledger.record(_ledger.MV_DOT, flops=2 * m)
            alpha = float(np.sqrt(nrm2))
            self._guard_alpha(alpha, self._wscale)
            e.divide_into(e.col(j), self._w, alpha)
            self._emit_host(self._s + c, alpha)
            self._pending = False
            self._s = None
        return super().finalize()


_STATES = {cls.scheme_id: cls for cls in (Cgs2State, Dcgs2State)}


def make_state(scheme, m, n_cap, ledger=None, **options):
    """Construct the push state for a scheme id (ortho.py:483-489)."""
    if scheme not in _STATES:
        raise UnknownSchemeError(
            f"unknown scheme {scheme!r} (the B200 backend provides {', '.join(SCHEME_IDS)})")
    return _STATES[scheme](m, n_cap, ledger=ledger, **options)


def qr_factorize(A, scheme, ledger=None, **options):
    """Factorize a tall matrix column by column; returns (Q, R)
    (ortho.py:492-507).  A is a host array (m, n) or a device tensor of this
    rank's rows."""
    if isinstance(A, torch.Tensor) and A.is_cuda:
        if A.dim() != 2:
            raise DimensionError(f"tall matrix expected, got {tuple(A.shape)}")
        n = A.shape[1]
        m = int(options.pop("m_global", A.shape[0]))
        cols = [A[:, j].contiguous() for j in range(n)]
    else:
        A = np.asarray(A, dtype=np.float64)
        if A.ndim != 2 or A.shape[0] < A.shape[1]:
            raise DimensionError(f"tall matrix expected, got {A.shape}")
        m, n = A.shape
        cols = None
    if m < n:
        raise DimensionError(f"tall matrix expected, got {(m, n)}")
    state = make_state(scheme, m, n, ledger=ledger, **options)
    if cols is None:
        lo, hi = state.space.row_lo, state.space.row_hi
        dev = runtime.upload(np.asfortranarray(A[lo:hi]).T.copy())  # row c = column c
        cols = [dev[j] for j in range(n)]
    for j in range(n):
        state.push(cols[j])
    return state.finalize()
