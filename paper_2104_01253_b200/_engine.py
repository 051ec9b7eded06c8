"""Per-expansion device engine: one basis block, one stream, one reduction
workspace, one pinned result buffer, and the communicator of the operator.

Every reducing call is: kernel -> (allreduce over ranks) -> the reduced
scalars on the host.  On one GPU the reducing kernel's last CTA writes its
2j+3 results straight into page-locked host memory (device-mapped), so the
only host action per step is one stream synchronize; the update's
coefficients ride in the kernel launch (kls_*_host).  That is the single
host synchronization of a DCGS2 step.

The engine binds the stream that is current when it is created.
"""

import ctypes

import numpy as np
import torch

from . import _lib, runtime, trace
from .errors import DimensionError

_PACK = 2048  # coefficients that fit in a kernel launch (kls_*_host)


def _panels(j):
    """Column panels (of <= 256) a Gram launch with j basis columns runs as;
    each fused peer exchange consumes one epoch."""
    return max(1, -(-j // 256))


def _mapped(host_ptr):
    """Device address of a page-locked host address (identical under UVA)."""
    dptr = ctypes.c_void_p()
    try:
        _lib.call("kls_host_device_ptr", host_ptr, ctypes.byref(dptr))
        return dptr.value
    except _lib.KlsGpuError:
        return host_ptr


class Engine:
    def __init__(self, op, capacity):
        self.op = op
        self.comm = op.comm
        self.world = op.comm.world
        self.m = op.shape[0]  # global rows (guards, ledger flops)
        self.ml = op.m_local
        self.ld = runtime.pad_rows(self.ml)
        self.capacity = capacity
        dev = runtime.device()
        _lib.load()
        self.st = runtime.stream_handle()
        # column-major basis: row c of the buffer is column c of Q.  Not
        # zero-filled (a 100 GB memset per expansion): columns are written
        # before they are read, and zero_col() pads a breakdown column.
        self.vbuf = torch.empty((capacity, self.ld), dtype=torch.float64, device=dev)
        self.qptr = self.vbuf.data_ptr()
        nres = 2 * capacity + 8
        self.nres = nres
        self.stage = runtime.Staging(nres)
        # pinned result buffer the reducing kernels write into directly; the
        # second half is the other slot of the lookahead double buffer
        self.res_host = torch.zeros(3 * nres, dtype=torch.float64, pin_memory=True)
        self.res_np = self.res_host.numpy()[:nres]
        self.res_dev = _mapped(self.res_host.data_ptr())
        self.slot_np = [self.res_host.numpy()[nres * (1 + s) : nres * (2 + s)] for s in (0, 1)]
        self.slot_dev = [self.res_dev + 8 * nres * (1 + s) for s in (0, 1)]
        self.gdev = torch.empty(nres, dtype=torch.float64, device=dev)
        self.cdev = torch.empty(nres, dtype=torch.float64, device=dev)
        # completion events of the two lookahead slots (CUDA events owned by
        # the library, so kls_dcgs2_queue_step can record them too)
        self.slot_ev = []
        for _ in range(2):
            ev = ctypes.c_void_p()
            _lib.call("kls_event_create", ctypes.byref(ev))
            self.slot_ev.append(ev.value)
        self._plan = None  # kls_dcgs2_queue_step plan (one GPU), False when n/a
        self.ws, self.wsb = runtime.workspace_for(self.st, capacity + 1)
        # the rows' reduction layout (rank-count-independent segment tree)
        self.segs = op.segs
        self.segp = op.segs.ptr
        # N > 1: the per-step reduction goes over NVLink peer memory when
        # available (csrc/comm.cu), else through NCCL
        self.peer = runtime.peer_link(self.comm) if self.world > 1 else None

    # -- views ----------------------------------------------------------------
    def zero_col(self, c):
        if c < self.capacity:
            self.vbuf[c].zero_()

    def col(self, c):
        return self.vbuf[c, : self.ml]

    def block(self, k):
        """(m_local, k) column-major view of the first k columns."""
        return self.vbuf[:k, : self.ml].T

    # -- reductions -----------------------------------------------------------
    def _out(self, count):
        """Where a reducing kernel writes `count` results (world > 1: this
        rank's exported tree nodes, up to 8 x count)."""
        if self.world == 1:
            if count > self.res_np.size:
                raise DimensionError("result buffer too small")
            return self.res_dev
        self.stage.ensure(runtime.SEG_MAX_EXPORT * count)
        return self.stage.dev_out.data_ptr()

    def _combine_into(self, count, dst_ptr, dst=None):
        """world > 1: combine the exported nodes in stage.dev_out over the
        ranks into dst_ptr (peer exchange) or dst (NCCL path, a tensor)."""
        rec = trace._active
        if self.peer is not None:
            if count > self.res_np.size:
                raise DimensionError("result buffer too small")
            if rec is not None and rec.events:
                with rec.span("allreduce"):
                    self.peer.seg_combine(self.stage.dev_out.data_ptr(), count, dst_ptr, self.st)
            else:
                self.peer.seg_combine(self.stage.dev_out.data_ptr(), count, dst_ptr, self.st)
            return None
        if rec is not None and rec.events:
            with rec.span("allreduce"):
                out = self.comm.combine_(self.stage.dev_out, count)
        else:
            out = self.comm.combine_(self.stage.dev_out, count)
        if dst is not None:
            dst[:count].copy_(out)
        return out

    def _finish(self, count):
        if self.world == 1:
            _lib.call("kls_stream_sync", self.st)
            runtime.XFER["d2h"] += 8 * count
            return self.res_np[:count].copy()
        if self.peer is not None:
            self._combine_into(count, self.res_dev)
            _lib.call("kls_stream_sync", self.st)
            self.peer.check()
            runtime.XFER["d2h"] += 8 * count
            return self.res_np[:count].copy()
        out = self._combine_into(count, None)
        self.stage.dev_out[:count].copy_(out)
        return self.stage.fetch(count)

    def gram_dcgs2(self, j, w, aw):
        """[Q(:,0:j), w]^T [w, aw] and aw.aw over all ranks: 2j+3 values."""
        if self.peer is not None and 2 * j + 3 <= self.res_np.size:
            return self._gram_dcgs2_fused(j, w, aw)
        out = self._out(2 * j + 3)
        rec = trace._active
        if rec is None:
            _lib.call("kls_gram_dcgs2", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                      aw.data_ptr(), out, self.segp, self.ws, self.wsb, self.st)
        else:
            rec.note("gram", 8 * self.ml * (j + 2))
            with rec.span("gram"):
                _lib.call("kls_gram_dcgs2", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                          aw.data_ptr(), out, self.segp, self.ws, self.wsb, self.st)
        return self._finish(2 * j + 3)

    def _gram_dcgs2_fused(self, j, w, aw):
        """N > 1: Gram + one-shot NVLink allreduce in one kernel; the global
        sum lands in the mapped result buffer."""
        link = self.peer
        first = link.take_epochs(_panels(j))
        args = ("kls_gram_dcgs2_peer", self.qptr, self.ld, self.ml, j, w.data_ptr(), aw.data_ptr(),
                self.res_dev, self.segp, self.ws, self.wsb, link.ptrs, link.rank, link.world,
                link.CAP, first, link.err_dev, self.st)
        rec = trace._active
        if rec is None:
            _lib.call(*args)
        else:
            rec.note("gram", 8 * self.ml * (j + 2))
            with rec.span("gram"):
                _lib.call(*args)
        link.comm.allreduce_calls += 1
        _lib.call("kls_stream_sync", self.st)
        link.check()
        runtime.XFER["d2h"] += 8 * (2 * j + 3)
        return self.res_np[: 2 * j + 3].copy()

    # -- one-step lookahead --------------------------------------
    def gram_ahead(self, j, w, aw, slot, qr=False):
        """Queue Gram_j (+ the cross-rank reduction) and the device scalar
        step; the reduced vector lands in mapped slot `slot`, the update
        coefficients in self.cdev.  Nothing waits."""
        count = 2 * j + 3
        rec = trace._active
        if rec is not None:
            rec.note("gram", 8 * self.ml * (j + 2))
        fused = True  # scalar step fused into the Gram kernel's finishing CTA
        qflag = 1 if qr else 0
        if self.peer is not None:
            link = self.peer
            first = link.take_epochs(_panels(j))
            link.comm.allreduce_calls += 1
            args = ("kls_gram_dcgs2_peer_step", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                    aw.data_ptr(), self.gdev.data_ptr(), self.cdev.data_ptr(), self.slot_dev[slot],
                    qflag, self.segp, self.ws, self.wsb, link.ptrs, link.rank, link.world,
                    link.CAP, first, link.err_dev, self.st)
        elif self.world == 1:
            args = ("kls_gram_dcgs2_step", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                    aw.data_ptr(), self.gdev.data_ptr(), self.cdev.data_ptr(), self.slot_dev[slot],
                    qflag, self.segp, self.ws, self.wsb, self.st)
        else:
            fused = False
            dst = self.gdev.data_ptr() if self.world == 1 else self._out(count)
            args = ("kls_gram_dcgs2", self.qptr, self.ld, self.ml, j, w.data_ptr(), aw.data_ptr(),
                    dst, self.segp, self.ws, self.wsb, self.st)
        if rec is not None and rec.events:
            with rec.span("gram"):
                _lib.call(*args)
        else:
            _lib.call(*args)
        if not fused:
            if self.world > 1:
                self._combine_into(count, self.gdev.data_ptr(), self.gdev)
            _lib.call("kls_dcgs2_scalars", self.gdev.data_ptr(), j, qflag, self.cdev.data_ptr(),
                      self.slot_dev[slot], self.st)
        _lib.call("kls_event_record", self.slot_ev[slot], self.st)

    def wait_slot(self, slot, count):
        """Block until the queued Gram of `slot` has landed; its 2j+3 values."""
        _lib.call("kls_event_sync", self.slot_ev[slot])
        if self.peer is not None:
            self.peer.check()
        runtime.XFER["d2h"] += 8 * count
        return self.slot_np[slot][:count].copy()

    def update_ahead(self, j, w, w_out, aw, divide):
        """The fused update with the device-computed coefficients; w' goes
        to w_out (w stays intact)."""
        rec = trace._active
        if rec is not None:
            rec.note("update", 8 * self.ml * (j + 4))
        args = ("kls_dcgs2_update_dev", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                w_out.data_ptr(), aw.data_ptr(), self.cdev.data_ptr(), 1 if divide else 0,
                self.segp, self.st)
        if rec is not None and rec.events:
            with rec.span("update"):
                _lib.call(*args)
        else:
            _lib.call(*args)

    def project(self, k, x, xnorm=True):
        """Q(:,0:k)^T x (and x.x) over all ranks: k (+1) values."""
        n = k + (1 if xnorm else 0)
        if n == 0:
            return np.zeros(0)
        out = self._out(n)
        args = ("kls_mv_trans_mv", self.qptr if k else None, self.ld, self.ml, k, None,
                x.data_ptr(), None, 1, 1 if xnorm else 0, out, self.segp, self.ws, self.wsb,
                self.st)
        rec = trace._active
        if rec is None:
            _lib.call(*args)
        else:
            rec.note("project", 8 * self.ml * (k + 1))
            with rec.span("project"):
                _lib.call(*args)
        return self._finish(n)

    def sqnorm(self, x):
        return float(self.project(0, x, xnorm=True)[0])

    # -- updates ----------------------------------------------------------------
    def dcgs2_update(self, j, w, aw, c, t, alpha, divide):
        coef = np.concatenate([c, t])
        rec = trace._active
        if rec is not None:
            rec.note("update", 8 * self.ml * (j + 4))
        if coef.size <= _PACK:
            runtime.XFER["h2d"] += 8 * coef.size
            args = ("kls_dcgs2_update_host", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                    aw.data_ptr(), coef.ctypes.data, float(alpha), 1 if divide else 0, self.segp,
                    self.st)
        else:
            dev = self.stage.push(coef)
            args = ("kls_dcgs2_update", self.qptr, self.ld, self.ml, j, w.data_ptr(),
                    aw.data_ptr(), dev.data_ptr(), float(alpha), 1 if divide else 0, self.segp,
                    self.st)
        if rec is not None and rec.events:
            with rec.span("update"):
                _lib.call(*args)
        else:
            _lib.call(*args)

    def subtract_projection(self, y, k, coef, want_norm=False):
        """y <- y - Q(:,0:k) coef; optionally return ||y||^2 over all ranks."""
        nrm = self._out(1) if want_norm else None
        if k <= _PACK:
            c = np.ascontiguousarray(coef, dtype=np.float64) if k else None
            runtime.XFER["h2d"] += 8 * k
            args = ("kls_mv_times_mat_add_mv_host", y.data_ptr(), self.ld, self.ml, 1,
                    self.qptr if k else None, self.ld, k, c.ctypes.data if k else None,
                    -1.0, 1.0, nrm, self.segp, self.ws, self.wsb, self.st)
        else:
            dev = self.stage.push(coef)
            args = ("kls_mv_times_mat_add_mv", y.data_ptr(), self.ld, self.ml, 1, self.qptr,
                    self.ld, k, dev.data_ptr(), -1.0, 1.0, nrm, self.segp, self.ws, self.wsb,
                    self.st)
        rec = trace._active
        if rec is None:
            _lib.call(*args)
        else:
            rec.note("mtm", 8 * self.ml * (k + 2))
            with rec.span("mtm"):
                _lib.call(*args)
        if want_norm:
            return float(self._finish(1)[0])
        return None

    def subtract_and_project(self, y, k, coef):
        """y <- y - Q(:,0:k) coef, then Q(:,0:k)^T y over all ranks: CGS2's
        first update and second projection in one pass (kls_project_gram)."""
        if k == 0:
            return np.zeros(0)
        if k > _PACK:
            self.subtract_projection(y, k, coef)
            return self.project(k, y, xnorm=False)
        c = np.ascontiguousarray(coef, dtype=np.float64)
        runtime.XFER["h2d"] += 8 * k
        args = ("kls_project_gram", self.qptr, self.ld, self.ml, k, y.data_ptr(), c.ctypes.data,
                1, 0, self._out(k), self.segp, self.ws, self.wsb, self.st)
        rec = trace._active
        if rec is None:
            _lib.call(*args)
        else:
            rec.note("project_gram", 8 * self.ml * (k + 2))
            with rec.span("project_gram"):
                _lib.call(*args)
        return self._finish(k)

    def _reduce_into(self, count, launch, dst):
        """Queue a reducing kernel whose `count` global results go to the
        device tensor `dst` (world 1: written directly; otherwise exported
        tree nodes, then the cross-rank combine) -- nothing waits."""
        if self.world == 1:
            launch(dst.data_ptr())
            return
        launch(self._out(count))
        self._combine_into(count, dst.data_ptr(), dst)

    def cgs2_chain(self, j, v):
        """Cgs2State.push's three reductions for column v against Q(:, 0:j),
        chained on the device with ONE host wait: s = Q^T v and v.v
        (kls_mv_trans_mv), v <- v - Q s and c = Q^T v with s read from the
        device (kls_project_gram), v <- v - Q c and ||v||^2 (the fused-norm
        update, c from the device).  Each reduction is still a separate
        global reduction (3 per step, the comparator's cost model); only the
        host round trips between them are gone.  Returns host (s, ||v0||^2,
        c, ||v||^2)."""
        n1 = j + 1
        g = self.gdev
        rec = trace._active
        gp = g.data_ptr()

        def span(name, nbytes, fn):
            if rec is None:
                fn()
            else:
                rec.note(name, nbytes)
                with rec.span(name):
                    fn()

        span("project", 8 * self.ml * (j + 1), lambda: self._reduce_into(n1, lambda o: _lib.call(
            "kls_mv_trans_mv", self.qptr, self.ld, self.ml, j, None, v.data_ptr(), None, 1, 1, o,
            self.segp, self.ws, self.wsb, self.st), g[:n1]))
        span("project_gram", 8 * self.ml * (j + 2), lambda: self._reduce_into(j, lambda o: _lib.call(
            "kls_project_gram", self.qptr, self.ld, self.ml, j, v.data_ptr(), gp, 0, 0, o,
            self.segp, self.ws, self.wsb, self.st), g[n1 : n1 + j]))
        span("mtm", 8 * self.ml * (j + 2), lambda: self._reduce_into(1, lambda o: _lib.call(
            "kls_mv_times_mat_add_mv", v.data_ptr(), self.ld, self.ml, 1, self.qptr, self.ld, j,
            gp + 8 * n1, -1.0, 1.0, o, self.segp, self.ws, self.wsb, self.st), g[n1 + j : n1 + j + 1]))
        cnt = 2 * j + 2
        h = self.stage.host_out[:cnt]
        h.copy_(g[:cnt], non_blocking=True)
        _lib.call("kls_stream_sync", self.st)
        if self.peer is not None:
            self.peer.check()
        runtime.XFER["d2h"] += 8 * cnt
        r = h.numpy().copy()
        return r[:j], float(r[j]), r[n1 : n1 + j], float(r[n1 + j])

    def add_combination(self, y, x, k, coef):
        """y = x + Q(:, 0:k) coef (host coefficients ride in the launch)."""
        if y.data_ptr() != x.data_ptr():
            y.copy_(x)
        if k == 0:
            return
        c = np.ascontiguousarray(coef[:k], dtype=np.float64)
        trace.note("mtm", 8 * self.ml * (k + 2))
        if k <= _PACK:
            _lib.call("kls_mv_times_mat_add_mv_host", y.data_ptr(), self.ld, self.ml, 1, self.qptr,
                      self.ld, k, c.ctypes.data, 1.0, 1.0, None, None, self.ws, self.wsb,
                      self.st)
        else:
            dev = self.stage.push(c)
            _lib.call("kls_mv_times_mat_add_mv", y.data_ptr(), self.ld, self.ml, 1, self.qptr,
                      self.ld, k, dev.data_ptr(), 1.0, 1.0, None, None, self.ws, self.wsb,
                      self.st)

    def resid_norms(self, b, ax, x):
        """[||b - ax||^2, ||x||^2, ||b||^2] over all ranks, one pass."""
        out = self._out(3)
        trace.note("resid_norms", 24 * self.ml)
        _lib.call("kls_resid_norms", b.data_ptr(), ax.data_ptr(), x.data_ptr(), self.ml, out,
                  self.segp, self.ws, self.wsb, self.st)
        return self._finish(3)

    def resid_norms_queue(self, b, ax, x, out):
        """resid_norms into the device tensor `out` (3 doubles, combined over
        ranks) without waiting: for diagnostics read back later in bulk."""
        trace.note("resid_norms", 24 * self.ml)
        if self.world == 1:
            _lib.call("kls_resid_norms", b.data_ptr(), ax.data_ptr(), x.data_ptr(), self.ml,
                      out.data_ptr(), self.segp, self.ws, self.wsb, self.st)
            return
        _lib.call("kls_resid_norms", b.data_ptr(), ax.data_ptr(), x.data_ptr(), self.ml,
                  self._out(3), self.segp, self.ws, self.wsb, self.st)
        self._combine_into(3, out.data_ptr(), out)

    def divide_into(self, dst, src, alpha):
        trace.note("scale", 16 * self.ml)
        _lib.call("kls_scale", src.data_ptr(), dst.data_ptr(), self.ml, float(alpha), 0, self.st)

    # -- operator -----------------------------------------------------------------
    def apply(self, x, y):
        """Uncounted operator application (the caller bumps op.napply)."""
        self.op.apply_into(x, y, self.st)

    def apply_resid_norms(self, x, y, b, out):
        """GMRES's backward-error column (gmres.py:171-172): y = A x and the
        norms [||b - y||^2, ||x||^2, ||b||^2] into the device tensor `out`,
        without waiting.  On one GPU with an ELL operator the two are one
        kernel (kls_ell_resid_norms: A x bit-identical, y not stored);
        otherwise the product and kls_resid_norms."""
        ell = getattr(self.op, "_ell", None)
        if (self.world == 1 and ell is not None and trace._active is None
                and not getattr(self.op, "_peer", False)):
            ecol, evals, elen, width, ld = ell
            _lib.call("kls_ell_resid_norms", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(),
                      width, self.ml, ld, x.data_ptr(), b.data_ptr(), out.data_ptr(), self.segp,
                      self.ws, self.wsb, self.st)
            return
        self.apply(x, y)
        self.resid_norms_queue(b, y, x, out)

    def __del__(self):
        try:
            for ev in getattr(self, "slot_ev", ()):
                _lib.call("kls_event_destroy", ev)
        except Exception:  # interpreter shutdown: the driver reclaims them
            pass

    # -- one-GPU step plan (kls_dcgs2_queue_step) ---------------------------------
    def step_plan(self, qr=False):
        """The launch plan of the lookahead step — update, operator, Gram +
        scalar step, slot event — as one host call, or None (several ranks,
        an operator without a plain-pointer description, or a tracer that
        times each kernel)."""
        if trace._active is not None:
            return None
        if self._plan is None:
            self._plan = False
            desc = self.op.op_desc() if self.world == 1 else None
            if desc is not None:
                p = _lib.KlsStepPlan()
                p.Q, p.ldq, p.m = self.qptr, self.ld, self.ml
                p.segs = self.segs.c
                p.gdev, p.cdev = self.gdev.data_ptr(), self.cdev.data_ptr()
                p.gout[0], p.gout[1] = self.slot_dev
                p.ws, p.ws_bytes, p.stream = self.ws, self.wsb, self.st
                p.event[0], p.event[1] = self.slot_ev
                p.divide, p.qr = (0, 1) if qr else (1, 0)
                p.op = desc
                self._plan = p
        return self._plan or None

    def queue_step(self, plan, j, w, w_out, aw, aw_out, slot, gram):
        """Step j of the lookahead through the plan: w -> w_out (and column j),
        A w_out -> aw_out, then (gram) Gram_{j+1} into `slot`."""
        _lib.call("kls_dcgs2_queue_step", ctypes.byref(plan), j, w.data_ptr(), w_out.local.data_ptr(),
                  w_out.ext_ptr, aw.data_ptr(), aw_out.data_ptr(), slot, 1 if gram else 0)
        _lib.count_launches(2 if gram else 1)

    def queue_step_be(self, plan, j, w, w_out, aw, aw_out, slot, gram, job):
        """queue_step with a GMRES backward-error column riding on it
        (kls_dcgs2_queue_step_be): job = (x, xj, axj, y, b, out) computes
        xj = x + Q(:, 0:len(y)) y and out = [||b - A xj||^2, ||xj||^2,
        ||b||^2] inside the step's update and ELL product."""
        x, xj, _, y, b, out = job
        yc = np.ascontiguousarray(y, dtype=np.float64)
        be = _lib.KlsBeCol(x=x.data_ptr(), xj=xj.data_ptr(), q=len(yc), y=yc.ctypes.data,
                           b=b.data_ptr(), out=out.data_ptr())
        trace.note("mtm", 16 * self.ml)
        _lib.call("kls_dcgs2_queue_step_be", ctypes.byref(plan), j, w.data_ptr(),
                  w_out.local.data_ptr(), w_out.ext_ptr, aw.data_ptr(), aw_out.data_ptr(), slot,
                  1 if gram else 0, ctypes.byref(be))
        _lib.count_launches(2 if gram else 1)

    def be_fusable(self):
        """Whether a GMRES backward-error column can ride on a lookahead step
        (one rank, the step plan, an ELL operator)."""
        plan = self.step_plan()
        return plan is not None and plan.op.kind == _lib.OP_ELL

    def check_capacity(self, n):
        if n > self.capacity:
            raise DimensionError("expansion capacity exhausted")
