"""Arnoldi expansions A V_k = V_{k+1} Hbar_k on the device (reference
arnoldi.py).

The basis V lives in HBM (column-major, one padded column per basis
vector); the small Hessenberg matrix and the DCGS2 correction ledger K stay
on the host in numpy, updated in exactly the reference's order from the
reduced Gram scalars, so H is bit-faithful to the scalars it is given.

``dcgs2`` — _DelayedArnoldi (arnoldi.py:307-455): one fused reduction per
step (kls_gram_dcgs2), one fused update pass (kls_dcgs2_update), one
operator application.  ``cgs2`` — _ImmediateArnoldi with CGS2
(arnoldi.py:121-172, ortho.py:139-158): three reductions per step.
Other reference schemes are outside the hot path and
raise UnknownSchemeError.
"""

import ctypes
import os

import numpy as np
import torch

from . import _lib, runtime
from . import ledger as _ledger
from ._engine import Engine
from .errors import BreakdownError, DimensionError, UnknownSchemeError
from .ledger import SyncLedger

_EPS = np.finfo(np.float64).eps

ARNOLDI_SCHEMES = ("cgs2", "dcgs2")


def _unsupported(scheme):
    return UnknownSchemeError(
        f"unknown scheme {scheme!r} (the B200 backend provides {', '.join(ARNOLDI_SCHEMES)})")


_HOST_BLAS = None  # (cblas_ddot, cblas_dgemv) of numpy's OpenBLAS, or False


def _host_blas():
    """numpy's own OpenBLAS entry points (ILP64 scipy-openblas), so the C++
    host step (kls_dcgs2_host_step) reproduces numpy's dot / matmul bit for
    bit; False (numpy path) when this numpy carries another BLAS or the C++
    step fails its self-check against the numpy step."""
    global _HOST_BLAS
    if _HOST_BLAS is None:
        _HOST_BLAS = False
        try:
            import ctypes
            import glob

            libs = glob.glob(os.path.join(os.path.dirname(np.__file__), os.pardir, "numpy.libs",
                                          "libscipy_openblas64_*.so"))
            if len(libs) == 1:
                blas = ctypes.CDLL(libs[0])
                fns = (ctypes.cast(blas.scipy_cblas_ddot64_, ctypes.c_void_p).value,
                       ctypes.cast(blas.scipy_cblas_dgemv64_, ctypes.c_void_p).value)
                if _host_step_selfcheck(fns):
                    _HOST_BLAS = fns
        except (OSError, AttributeError):
            _HOST_BLAS = False
    return _HOST_BLAS


def _host_step_c(g, j, m, wscale, k_prev, h, blas):
    t_full = np.empty(j + 1)
    k_next = np.empty(j + 1)
    res = np.empty(2)
    kp = np.ascontiguousarray(k_prev, dtype=np.float64) if j > 0 else None
    st = _lib.load().kls_dcgs2_host_step(
        g.ctypes.data, j, m, float(wscale), kp.ctypes.data if kp is not None else None,
        h.ctypes.data, h.shape[1], t_full.ctypes.data, k_next.ctypes.data, res.ctypes.data,
        blas[0], blas[1])
    return st, t_full, k_next, res


def _host_step_selfcheck(blas):
    """The C++ step against the numpy step on seeded inputs: bitwise."""
    rng = np.random.default_rng(5)
    for j in (0, 1, 2, 7, 33, 100):
        cap = j + 3
        g = np.ascontiguousarray(rng.standard_normal(2 * j + 3))
        g[j] = float(g[:j] @ g[:j]) + 4.0
        g[2 * j + 2] = abs(g[2 * j + 2])
        k_prev = rng.standard_normal(j)
        h1 = rng.standard_normal((cap, cap - 1))
        h2 = h1.copy()
        ref = _host_step_numpy(g, j, 1000, 0.5, k_prev, h1, SyncLedger())
        st, t_full, k_next, res = _host_step_c(g, j, 1000, 0.5, k_prev, h2, blas)
        if st != 0 or ref is None:
            return False
        if not (np.array_equal(h1, h2) and np.array_equal(ref[1], t_full)
                and np.array_equal(ref[4], k_next) and ref[2] == res[0] and ref[3] == res[1]):
            return False
    return True


def dcgs2_host_step(g, j, m, wscale, k_prev, h, ledger):
    """Host half of a DCGS2 step (arnoldi.py:367-420); see _host_step_numpy.
    Runs in C++ (kls_dcgs2_host_step) with numpy's own BLAS when available —
    identical bits, a fraction of the Python overhead."""
    blas = _host_blas()
    if not blas or h.dtype != np.float64 or not h.flags.c_contiguous:
        return _host_step_numpy(g, j, m, wscale, k_prev, h, ledger)
    g = np.ascontiguousarray(g, dtype=np.float64)
    st, t_full, k_next, res = _host_step_c(g, j, m, wscale, k_prev, h, blas)
    if st == 1:
        return None
    if st == 2:
        ledger.add_flops(2 * j)  # the c.c of the failed norm, as the numpy step
        raise BreakdownError(f"cancellation in the delayed norm of basis column {j}",
                             kind="pythagorean", column=j)
    if st != 0:
        raise RuntimeError("kls_dcgs2_host_step: bad arguments")
    ledger.add_flops(2 * j)
    ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * j)  # u = w - Q c
    ledger.add_flops(2 * j)
    ledger.add_flops(2 * (j + 1) * j)
    ledger.add_flops(m)
    ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * (j + 1))  # w' = aw/alpha - V t
    return g[:j].copy(), t_full, float(res[0]), float(res[1]), k_next


def _host_step_numpy(g, j, m, wscale, k_prev, h, ledger):
    """Host half of a DCGS2 Arnoldi step (arnoldi.py:367-420), from the
    reduced vector g = [c, beta, s, s_piv, ||aw||^2] of kls_gram_dcgs2.

    Runs identically on every rank (the allreduced g is bitwise the same on
    all of them), so no broadcast is needed.  Completes Hessenberg column
    j-1 in ``h`` in the reference's order.  Returns None on a happy
    breakdown, else (c, t_full, alpha, vscale, K_next) for the fused update.
    Raises BreakdownError("pythagorean") like the reference.
    """
    c = np.array(g[:j], dtype=np.float64)
    beta = float(g[j])
    s = np.array(g[j + 1 : 2 * j + 1], dtype=np.float64)
    s_piv = float(g[2 * j + 1])
    aw_norm = float(np.sqrt(g[2 * j + 2]))
    if not np.sqrt(max(beta, 0.0)) > _EPS * np.sqrt(m) * wscale:
        if j > 0:
            h[:j, j - 1] = k_prev + c
            h[j, j - 1] = 0.0
        return None
    alpha_sq = beta - float(c @ c)
    ledger.add_flops(2 * j)
    if not alpha_sq > beta * _EPS * _EPS:
        raise BreakdownError(f"cancellation in the delayed norm of basis column {j}",
                             kind="pythagorean", column=j)
    alpha = float(np.sqrt(alpha_sq))
    ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * j)  # u = w - Q c
    t_piv = (s_piv - float(c @ s)) / (alpha * alpha)
    ledger.add_flops(2 * j)
    t_full = np.empty(j + 1)
    np.divide(s, alpha, out=t_full[:j])
    t_full[j] = t_piv
    if j > 0:
        h[:j, j - 1] = k_prev + c
        h[j, j - 1] = alpha
    hc = h[: j + 1, :j] @ c
    ledger.add_flops(2 * (j + 1) * j)
    k_next = t_full - hc / alpha
    vscale = aw_norm / alpha  # pre-projection norm, arnoldi.py:414
    ledger.add_flops(m)
    ledger.record(_ledger.MV_TIMES_MAT_ADD_MV, flops=2 * m * (j + 1))  # w' = aw/alpha - V t
    return c, t_full, alpha, vscale, k_next


class _BaseArnoldi:
    scheme_id = None

    def __init__(self, op, capacity, ledger, engine=None):
        if capacity < 2:
            raise DimensionError("capacity of at least 2 basis vectors required")
        self.op = op
        self.capacity = capacity
        self.ledger = ledger if ledger is not None else SyncLedger()
        self.m = op.shape[0]
        # a caller (Krylov-Schur restart) may hand over an engine whose basis
        # buffer already holds the columns to resume from
        self.eng = engine if engine is not None else Engine(op, capacity)
        self._h = np.zeros((capacity, capacity - 1))
        self.nbasis = 0
        self.hcols = 0
        self.happy = False
        self.start_norm = None
        # a GMRES backward-error column to run inside the next lookahead step
        # (gmres.py sets it; _DelayedArnoldi._step_ahead runs it fused or,
        # without the step plan, separately -- either way exactly once)
        self._be_job = None

    def _run_be_job(self, job):
        """A GMRES backward-error column (x, x_j, scratch, y, b, out) through
        the separate launches: x_j = x + V y, then its norms."""
        if job is not None:
            x, xj, axj, y, b, out = job
            self.eng.add_combination(xj, x, len(y), y)
            self.eng.apply_resid_norms(xj, axj, b, out)

    # -- views (device tensors for the basis, numpy for H) -------------------------
    @property
    def basis(self):
        return self.eng.block(self.nbasis)

    @property
    def h(self):
        rows = min(self.hcols + 1, self.nbasis)
        return self._h[:rows, : self.hcols]

    @property
    def h_extended(self):
        return self._h[: self.hcols + 1, : self.hcols]

    @property
    def basis_extended(self):
        return self.eng.block(self.hcols + 1)

    @property
    def size(self):
        return self.nbasis + (1 if self._has_pending() else 0)

    @property
    def order(self):
        return self.size if self.happy else self.size - 1

    def _has_pending(self):
        return False

    # -- contract -----------------------------------------------------------------
    def step(self):
        """Grow by one column; False once a happy breakdown has been hit."""
        if self.happy:
            return False
        if self.size >= self.capacity:
            raise DimensionError("expansion capacity exhausted")
        return self._step()

    def finalize(self):
        """Flush pending work; returns (V, Hbar).

        V is an (m_local, nbasis) column-major view of the device basis (not a
        copy: at m = 1e8 a copy would double a 100 GB footprint; basis columns
        are append-only, so the view stays valid).  Hbar is a host copy.
        """
        self._flush()
        return self.eng.block(self.nbasis), self._h[: self.nbasis, : self.hcols].copy()

    def _step(self):
        raise NotImplementedError

    def _flush(self):
        pass

    def _mark_happy(self):
        # basis_extended shows one zero column past a breakdown (the
        # reference's zero-initialized storage)
        self.eng.zero_col(self.nbasis)
        self.happy = True
        return False

    def _load_basis(self, basis, ncols):
        e = self.eng
        e.check_capacity(ncols)
        if isinstance(basis, torch.Tensor) and basis.is_cuda:
            if basis.shape != (e.ml, ncols):
                raise DimensionError(f"basis of shape ({e.ml}, {ncols}) expected")
            e.vbuf[:ncols, : e.ml].copy_(basis.T)
        else:
            b = np.asarray(basis, dtype=np.float64)
            lo, hi = self.op.row_lo, self.op.row_hi
            if b.shape[0] == self.m and (hi - lo) != self.m:
                b = b[lo:hi]
            e.vbuf[:ncols, : e.ml].copy_(torch.from_numpy(np.ascontiguousarray(b.T)))

    # -- ledger helpers (global m, reference flop formulas) -------------------------
    def _rec(self, cls, flops):
        self.ledger.record(cls, flops=flops)


class _DelayedArnoldi(_BaseArnoldi):
    """One-reduction delayed reorthogonalization (dcgs2)."""

    scheme_id = "dcgs2"

    def __init__(self, op, start, capacity, ledger=None, engine=None):
        super().__init__(op, capacity, ledger, engine)
        e = self.eng
        self._w = op.new_vector()  # pending vector, with halo space
        self._aw = torch.zeros(e.ld, dtype=torch.float64, device=e.vbuf.device)[: e.ml]
        self._pending = False
        self._wscale = 0.0
        self._k = None
        # one-step lookahead: (slot,) of a queued Gram of the
        # current pending vector, or None
        self._lookahead = os.environ.get("KLS_LOOKAHEAD", "1") != "0"
        self._ahead = None
        self._slot = 0
        # the lookahead writes the next pending vector and its image into a
        # second pair of buffers, so a discarded step leaves w / aw intact
        self._w2 = self._aw2 = None
        if self._lookahead:
            self._w2 = op.new_vector()
            self._aw2 = torch.zeros(e.ld, dtype=torch.float64, device=e.vbuf.device)[: e.ml]
        if start is not None:
            self._w.local.copy_(op.take(start, "start vector"))
            nrm = float(np.sqrt(e.sqnorm(self._w.local)))  # local norm, not counted
            if not nrm > 0.0:
                raise ValueError("zero start vector")
            op.napply += 1
            e.apply(self._w, self._aw)
            self._pending = True
            self._wscale = nrm

    @classmethod
    def resume(cls, op, basis, hbar, capacity, ledger=None):
        self = cls(op, None, capacity, ledger)
        k = hbar.shape[1]
        self._load_basis(basis, k + 1)
        self._h[: k + 1, :k] = hbar
        self.nbasis = k + 1
        self.hcols = k
        return self

    def _has_pending(self):
        return self._pending

    def _step(self):
        e = self.eng
        m = self.m
        if not self._pending:
            # resumed without pending work: prime from the image of the last
            # (normalized) basis column (arnoldi.py:350-361)
            j = self.nbasis
            if getattr(self._w, "leased", True) is False:  # released by a finalize
                self._w = self.op.new_vector()
                if self._w2 is not None:
                    self._w2 = self.op.new_vector()
            w = self._w
            self.op.napply += 1
            e.apply(e.col(j - 1), w.local)
            r = e.project(j, w.local, xnorm=True)  # s = Q^T v, plus ||v||^2 (local)
            s, vnorm2 = r[:j].copy(), float(r[j])
            self._rec(_ledger.MV_TRANS_MV, 2 * m * j)
            e.subtract_projection(w.local, j, s)
            self._rec(_ledger.MV_TIMES_MAT_ADD_MV, 2 * m * j)
            self._k = s
            self.op.napply += 1
            e.apply(w, self._aw)
            self._pending = True
            self._wscale = float(np.sqrt(vnorm2))
            return True

        j = self.nbasis
        if self._lookahead:
            return self._step_ahead(j)
        g = e.gram_dcgs2(j, self._w.local, self._aw)
        self._rec(_ledger.MV_TRANS_MV, 2 * m * (j + 1) * 2)
        res = dcgs2_host_step(g, j, m, self._wscale, self._k, self._h, self.ledger)
        if j > 0:
            self.hcols = j
        if res is None:  # the pending direction vanished: invariant subspace
            self._pending = False
            return self._mark_happy()
        c, t_full, alpha, vscale, self._k = res
        if self.start_norm is None:
            self.start_norm = alpha
        # one pass: Q(:, j) = (w - Q c)/alpha; w = aw/alpha - Q t - q_j t_j
        e.dcgs2_update(j, self._w.local, self._aw, c, t_full, alpha, divide=True)
        self.nbasis += 1
        self.op.napply += 1
        e.apply(self._w, self._aw)
        self._wscale = vscale
        return True

    def _step_ahead(self, j):
        """The same step with a one-step lookahead: the update (with
        device-computed coefficients), the operator and the next Gram pass are
        queued before the host looks at this step's scalars, so the GPU never
        waits for the host.  The host then runs the reference's guards and H /
        K bookkeeping on the same scalars; on a breakdown the speculative work
        is discarded (it never touches finalized basis columns)."""
        e = self.eng
        m = self.m
        w, aw, w2, aw2 = self._w, self._aw, self._w2, self._aw2
        if self._ahead is None:
            e.gram_ahead(j, w.local, aw, self._slot)
        slot = self._slot
        # speculation: this step's update and operator (into the spare
        # buffers), then the next Gram
        nxt = 1 - slot if j + 2 < self.capacity else None
        self.op.napply += 1
        plan = e.step_plan()
        job, self._be_job = self._be_job, None
        if plan is not None and job is not None and plan.op.kind == _lib.OP_ELL:
            e.queue_step_be(plan, j, w.local, w2, aw, aw2, nxt or 0, nxt is not None, job)
        elif plan is not None:  # one host call for the three launches
            self._run_be_job(job)
            e.queue_step(plan, j, w.local, w2, aw, aw2, nxt or 0, nxt is not None)
        else:
            self._run_be_job(job)
            e.update_ahead(j, w.local, w2.local, aw, divide=True)
            e.apply(w2, aw2)
            if nxt is not None:
                e.gram_ahead(j + 1, w2.local, aw2, nxt)
        g = e.wait_slot(slot, 2 * j + 3)
        self._rec(_ledger.MV_TRANS_MV, 2 * m * (j + 1) * 2)
        try:
            res = dcgs2_host_step(g, j, m, self._wscale, self._k, self._h, self.ledger)
        except BreakdownError:
            self._ahead = None
            self.op.napply -= 1
            raise
        if j > 0:
            self.hcols = j
        if res is None:  # happy breakdown: drop the speculative column and apply
            self._ahead = None
            self.op.napply -= 1
            self._pending = False
            return self._mark_happy()
        _, _, alpha, vscale, self._k = res
        if self.start_norm is None:
            self.start_norm = alpha
        self.nbasis += 1
        self._wscale = vscale
        self._w, self._w2 = w2, w
        self._aw, self._aw2 = aw2, aw
        self._ahead = nxt
        if nxt is not None:
            self._slot = nxt
        return True

    def run_steps(self, nsteps):
        """Up to `nsteps` steps; the same results, ledger and exceptions as
        calling step() that often.  On one GPU with the step plan and the C++
        host step available the whole lookahead loop runs in one library call
        (kls_dcgs2_run); otherwise it is the step() loop."""
        done = 0
        while done < nsteps and not self.happy:
            if self.size >= self.capacity:
                raise DimensionError("expansion capacity exhausted")
            n = self._run_native(min(nsteps - done, self.capacity - self.size))
            if n is None:  # not eligible: one regular step
                if not self.step():
                    break
                n = 1
            done += n
            if n == 0:
                break
        return done

    def _run_native(self, nsteps):
        e = self.eng
        blas = _host_blas()
        if (not self._lookahead or not self._pending or nsteps < 2 or not blas
                or e.world != 1 or not self._h.flags.c_contiguous):
            return None
        plan = e.step_plan()
        if plan is None:
            return None
        j0 = self.nbasis
        w, aw, w2, aw2 = self._w, self._aw, self._w2, self._aw2
        if self._ahead is None:
            e.gram_ahead(j0, w.local, aw, self._slot)
        cap = self.capacity
        if getattr(self, "_run", None) is None:
            st = _lib.KlsRunState()
            st.plan = ctypes.pointer(plan)
            st.h, st.ldh = self._h.ctypes.data, self._h.shape[1]
            self._kbuf = np.zeros(cap)
            self._scratch = np.zeros(2 * cap)
            st.k, st.scratch = self._kbuf.ctypes.data, self._scratch.ctypes.data
            st.ddot, st.dgemv = blas
            st.m, st.capacity = self.m, cap
            st.gslot[0], st.gslot[1] = e.slot_np[0].ctypes.data, e.slot_np[1].ctypes.data
            self._run = st
        st = self._run
        st.w[0], st.w[1] = w.local.data_ptr(), w2.local.data_ptr()
        st.wx[0], st.wx[1] = w.ext_ptr, w2.ext_ptr
        st.aw[0], st.aw[1] = aw.data_ptr(), aw2.data_ptr()
        if j0 > 0:
            self._kbuf[:j0] = self._k
        io = np.zeros(7)
        io[0] = self._wscale
        _lib.call("kls_dcgs2_run", ctypes.byref(st), j0, nsteps, 0, self._slot, io.ctypes.data)
        done, status, jstop = int(io[2]), int(io[3]), int(io[4])
        queued = done + (1 if status else 0)
        _lib.count_launches(3 * queued)  # update, operator, Gram (+ scalar step)
        # the host read each step's 2j+3 scalars from mapped pinned memory
        jq = np.arange(j0, j0 + queued, dtype=np.int64)
        runtime.XFER["d2h"] += int(8 * np.sum(2 * jq + 3))
        m = self.m
        led = self.ledger
        js = np.arange(j0, j0 + done, dtype=np.int64)
        # the ledger of the completed steps (_step_ahead + dcgs2_host_step)
        led.record_many(_ledger.MV_TRANS_MV, done, int(np.sum(4 * m * (js + 1))))
        led.record_many(_ledger.MV_TIMES_MAT_ADD_MV, 2 * done,
                        int(np.sum(2 * m * js) + np.sum(2 * m * (js + 1))))
        led.add_flops(int(np.sum(4 * js + 2 * (js + 1) * js) + m * done))
        self.op.napply += done
        if done:
            self.nbasis += done
            jl = j0 + done - 1
            if jl > 0:
                self.hcols = jl
            if self.start_norm is None:
                self.start_norm = float(io[1])
            self._wscale = float(io[0])
            self._k = self._kbuf[: jl + 1].copy()
            if done % 2:
                self._w, self._w2 = w2, w
                self._aw, self._aw2 = aw2, aw
            nxt = int(io[5])
            self._ahead = nxt if nxt >= 0 else None
            if nxt >= 0:
                self._slot = nxt
        if status:
            # the breakdown step: its Gram reduction counted, its speculative
            # apply discarded (as _step_ahead)
            led.record(_ledger.MV_TRANS_MV, flops=4 * m * (jstop + 1))
            self._ahead = None
            if status == 2:
                led.add_flops(2 * jstop)
                raise BreakdownError(f"cancellation in the delayed norm of basis column {jstop}",
                                     kind="pythagorean", column=jstop)
            if jstop > 0:
                self.hcols = jstop
            self._pending = False
            self._mark_happy()
        return done

    def _release_w(self):
        for v in (self._w, self._w2):
            rel = getattr(v, "release", None)
            if rel is not None:
                rel()

    def _flush(self):
        """CGS2 pass on the pending vector (arnoldi.py:425-455): 2 reductions."""
        self._ahead = None  # a queued lookahead Gram of the pending vector is moot
        if not self._pending:
            self._release_w()
            return
        e = self.eng
        m = self.m
        j = self.nbasis
        w = self._w.local
        c = e.project(j, w, xnorm=False) if j else np.zeros(0)
        self._rec(_ledger.MV_TRANS_MV, 2 * m * j)
        nrm2 = e.subtract_projection(w, j, c, want_norm=True)  # u = w - Q c, ||u||^2
        self._rec(_ledger.MV_TIMES_MAT_ADD_MV, 2 * m * j)
        self._rec(_ledger.MV_DOT, 2 * m)
        alpha = float(np.sqrt(nrm2))
        if not alpha > _EPS * np.sqrt(m) * self._wscale:
            if j > 0:
                self._h[:j, j - 1] = self._k + c
                self._h[j, j - 1] = 0.0
                self.hcols = j
            self._pending = False
            self._mark_happy()
            self._release_w()
            return
        if self.start_norm is None:
            self.start_norm = alpha
        if j > 0:
            self._h[:j, j - 1] = self._k + c
            self._h[j, j - 1] = alpha
            self.hcols = j
        e.divide_into(e.col(j), w, alpha)
        self.nbasis += 1
        self._pending = False
        self._release_w()


class _ImmediateArnoldi(_BaseArnoldi):
    """CGS2 expansion: each column finished within its step (3 reductions)."""

    scheme_id = "cgs2"

    def __init__(self, op, start, capacity, ledger=None, engine=None):
        super().__init__(op, capacity, ledger, engine)
        e = self.eng
        self._v = torch.zeros(e.ld, dtype=torch.float64, device=e.vbuf.device)[: e.ml]
        # KLS_CGS2_CHAIN=0: one host round trip per reduction (round 1's path)
        self._chain = os.environ.get("KLS_CGS2_CHAIN", "1") != "0"
        self.last_coeffs = None
        self.last_alpha = None
        if start is not None:
            x = op.take(start, "start vector")
            nrm = float(np.sqrt(e.sqnorm(x)))  # local normalization, not counted
            if not nrm > 0.0:
                raise ValueError("zero start vector")
            self.start_norm = nrm
            e.divide_into(e.col(0), x, nrm)
            self.nbasis = 1

    @classmethod
    def resume(cls, op, basis, hbar, capacity, ledger=None):
        self = cls(op, None, capacity, ledger)
        k = hbar.shape[1]
        self._load_basis(basis, k + 1)
        self._h[: k + 1, :k] = hbar
        self.nbasis = k + 1
        self.hcols = k
        return self

    def _cgs2_push(self, v, j):
        """Cgs2State.push (ortho.py:144-158) of the device column v against
        Q(:, 0:j); returns (coeffs, alpha) and leaves u = v - Q(s+c) in v."""
        e = self.eng
        m = self.m
        if self._chain and j > 0:
            # the three reductions queued back to back on the device, one
            # host wait (Engine.cgs2_chain); the checks below then run in
            # the reference's order on the same scalars
            s, scale2, c, nrm2 = e.cgs2_chain(j, v)
            if not np.isfinite(scale2):
                raise ValueError("non-finite column")
            scale = float(np.sqrt(scale2))
            for kind in (_ledger.MV_TRANS_MV, _ledger.MV_TIMES_MAT_ADD_MV, _ledger.MV_TRANS_MV,
                         _ledger.MV_TIMES_MAT_ADD_MV):
                self._rec(kind, 2 * m * j)
            self._rec(_ledger.MV_DOT, 2 * m)
        else:
            r = e.project(j, v, xnorm=True)  # s = Q^T a and the local scale ||a||^2
            s, scale2 = r[:j].copy(), float(r[j])
            if not np.isfinite(scale2):
                raise ValueError("non-finite column")
            scale = float(np.sqrt(scale2))
            self._rec(_ledger.MV_TRANS_MV, 2 * m * j)
            c = e.subtract_and_project(v, j, s)  # one pass over Q for both
            self._rec(_ledger.MV_TIMES_MAT_ADD_MV, 2 * m * j)
            self._rec(_ledger.MV_TRANS_MV, 2 * m * j)
            nrm2 = e.subtract_projection(v, j, c, want_norm=True)
            self._rec(_ledger.MV_TIMES_MAT_ADD_MV, 2 * m * j)
            self._rec(_ledger.MV_DOT, 2 * m)
        alpha = float(np.sqrt(nrm2))
        self.last_coeffs, self.last_alpha = s + c, alpha
        if not alpha > _EPS * np.sqrt(m) * scale:
            raise BreakdownError(
                f"column {j} is dependent at working precision "
                f"(norm {alpha:.3e} against scale {scale:.3e})",
                kind="dependent", column=j)
        return s + c, alpha

    def _step(self):
        e = self.eng
        j = self.nbasis
        self.op.napply += 1
        e.apply(e.col(j - 1), self._v)
        try:
            coeffs, alpha = self._cgs2_push(self._v, j)
        except BreakdownError as err:
            if err.kind != "dependent":
                raise
            coeffs = self.last_coeffs
            self._h[: len(coeffs), j - 1] = coeffs
            self._h[j, j - 1] = 0.0
            self.hcols = j
            return self._mark_happy()
        self._h[: len(coeffs), j - 1] = coeffs
        self._h[j, j - 1] = alpha
        e.divide_into(e.col(j), self._v, alpha)
        self.nbasis += 1
        self.hcols = j
        return True


def arnoldi(op, start, scheme, capacity, ledger=None, **options):
    """Construct an expansion for a scheme id from a start vector
    (arnoldi.py:561-573)."""
    if options:
        raise TypeError(f"unexpected options {sorted(options)}")
    if scheme == "dcgs2":
        return _DelayedArnoldi(op, start, capacity, ledger)
    if scheme == "cgs2":
        return _ImmediateArnoldi(op, start, capacity, ledger)
    raise _unsupported(scheme)


def resume_arnoldi(op, basis, hbar, scheme, capacity, ledger=None, **options):
    """Continue from A V_k = V_{k+1} Hbar (arnoldi.py:576-600); the coupling
    row of hbar may be dense (Krylov-Schur form)."""
    if options:
        raise TypeError(f"unexpected options {sorted(options)}")
    hbar = np.asarray(hbar, dtype=np.float64)
    ncols = basis.shape[1]
    if ncols != hbar.shape[0] or hbar.shape[0] != hbar.shape[1] + 1:
        raise DimensionError(
            f"expected (m, k+1) basis with (k+1, k) hbar, got {tuple(basis.shape)} {hbar.shape}")
    if scheme == "dcgs2":
        return _DelayedArnoldi.resume(op, basis, hbar, capacity, ledger)
    if scheme == "cgs2":
        return _ImmediateArnoldi.resume(op, basis, hbar, capacity, ledger)
    raise _unsupported(scheme)


def arnoldi_expand(op, start, scheme, steps, ledger=None, **options):
    """Fixed-order expansion; returns (V, Hbar) (arnoldi.py:603-609)."""
    exp = arnoldi(op, start, scheme, capacity=steps + 1, ledger=ledger, **options)
    if hasattr(exp, "run_steps"):
        while exp.order < steps and not exp.happy:
            exp.run_steps(steps - exp.order)
    else:
        while exp.order < steps:
            if not exp.step():
                break
    return exp.finalize()
