"""Per-expansion device engine: one basis block, one stream, one reduction
workspace, one pinned staging pair, and the communicator of the operator.

Every reducing call here is: kernel -> (allreduce over ranks) -> one small
D2H of the reduced scalars.  That D2H is the only host synchronization of a
DCGS2 step.
"""

import numpy as np
import torch

from . import _lib, runtime, trace
from .errors import DimensionError


class Engine:
    def __init__(self, op, capacity):
        self.op = op
        self.comm = op.comm
        self.m = op.shape[0]  # global rows (guards, ledger flops)
        self.ml = op.m_local
        self.ld = runtime.pad_rows(self.ml)
        self.capacity = capacity
        dev = runtime.device()
        # column-major basis: row c of the buffer is column c of Q.  Not
        # zero-filled (a 100 GB memset per expansion): columns are written
        # before they are read, and zero_col() pads a breakdown column.
        self.vbuf = torch.empty((capacity, self.ld), dtype=torch.float64, device=dev)
        self.stage = runtime.Staging(2 * capacity + 8)
        runtime.workspace(capacity + 1)  # size it once up front

    @property
    def wsp(self):
        """(pointer, bytes) of the stream's reduction workspace."""
        return runtime.workspace(self.capacity + 1)

    def zero_col(self, c):
        if c < self.capacity:
            self.vbuf[c].zero_()

    # -- views ----------------------------------------------------------------
    def col(self, c):
        return self.vbuf[c, : self.ml]

    def block(self, k):
        """(m_local, k) column-major view of the first k columns."""
        return self.vbuf[:k, : self.ml].T

    @property
    def qptr(self):
        return self.vbuf.data_ptr()

    @property
    def st(self):
        return runtime.stream_handle()

    # -- reductions -----------------------------------------------------------
    def _finish(self, count):
        out = self.stage.dev_out[:count]
        if self.comm.world > 1:
            with trace.span("allreduce"):
                self.comm.allreduce_(out)
        return self.stage.fetch(count)

    def gram_dcgs2(self, j, w, aw):
        """[Q(:,0:j), w]^T [w, aw] and aw.aw over all ranks: 2j+3 values."""
        self.stage.ensure(2 * j + 3)
        ws, wsb = self.wsp
        trace.note("gram", 8 * self.ml * (j + 2))
        with trace.span("gram"):
            _lib.call("kls_gram_dcgs2", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                      aw.data_ptr(), self.stage.dev_out.data_ptr(), ws, wsb, self.st)
        return self._finish(2 * j + 3)

    def project(self, k, x, xnorm=True):
        """Q(:,0:k)^T x (and x.x) over all ranks: k (+1) values."""
        n = k + (1 if xnorm else 0)
        self.stage.ensure(max(n, 1))
        if n == 0:
            return np.zeros(0)
        ws, wsb = self.wsp
        trace.note("project", 8 * self.ml * (k + 1))
        _lib.call("kls_mv_trans_mv", self.qptr if k else None, self.ld, self.ml, k, None,
                  x.data_ptr(), None, 1, 1 if xnorm else 0, self.stage.dev_out.data_ptr(),
                  ws, wsb, self.st)
        return self._finish(n)

    def sqnorm(self, x):
        return float(self.project(0, x, xnorm=True)[0])

    # -- updates ----------------------------------------------------------------
    def dcgs2_update(self, j, w, aw, c, t, alpha, divide):
        coef = self.stage.push(np.concatenate([c, t]))
        trace.note("update", 8 * self.ml * (j + 4))
        with trace.span("update"):
            _lib.call("kls_dcgs2_update", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                      aw.data_ptr(), coef.data_ptr(), float(alpha), 1 if divide else 0, self.st)

    def subtract_projection(self, y, k, coef, want_norm=False):
        """y <- y - Q(:,0:k) coef; optionally return ||y||^2 over all ranks."""
        dev_coef = self.stage.push(coef) if k else None
        nrm = self.stage.dev_out.data_ptr() if want_norm else None
        ws, wsb = self.wsp
        trace.note("mtm", 8 * self.ml * (k + 2))
        _lib.call("kls_mv_times_mat_add_mv", y.data_ptr(), self.ld, self.ml, 1,
                  self.qptr if k else None, self.ld, k,
                  dev_coef.data_ptr() if k else None, -1.0, 1.0, nrm, ws, wsb, self.st)
        if want_norm:
            return float(self._finish(1)[0])
        return None

    def divide_into(self, dst, src, alpha):
        trace.note("scale", 16 * self.ml)
        _lib.call("kls_scale", src.data_ptr(), dst.data_ptr(), self.ml, float(alpha), 0, self.st)

    # -- operator -----------------------------------------------------------------
    def apply(self, x, y):
        """Uncounted operator application (the caller bumps op.napply)."""
        self.op.apply_into(x, y)

    def check_capacity(self, n):
        if n > self.capacity:
            raise DimensionError("expansion capacity exhausted")
