"""CPU oracle (numpy) for the DCGS2 / CGS2 Arnoldi-QR path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates the reference
algorithms of kls 0.1.0 (/root/reference/pkg/src/kls) with the same numpy
call shapes, so on the same BLAS it reproduces the reference to the last
bit; parity is pinned by tests/test_oracle.py against golden vectors the
reference itself produced (tests/golden/make_golden.py).

Citations are <file>:<line> in /root/reference/pkg/src/kls.
"""

from dataclasses import dataclass, field

import numpy as np

EPS = float(np.finfo(np.float64).eps)


class OracleBreakdown(RuntimeError):
    def __init__(self, msg, kind, column):
        super().__init__(msg)
        self.kind = kind
        self.column = column


@dataclass
class Counts:
    """Ledger-equivalent counters (ledger.py:23-62) plus operator applies."""

    reductions: int = 0
    flops: int = 0
    napply: int = 0
    kernels: dict = field(default_factory=lambda: {"MvTransMv": 0, "MvTimesMatAddMv": 0, "MvDot": 0})

    def rec(self, cls, flops=0):
        self.kernels[cls] += 1
        if cls != "MvTimesMatAddMv":
            self.reductions += 1
        self.flops += int(flops)


# ---------------------------------------------------------------------------
# operators


def csr_matvec(indptr, indices, data, x):
    """CsrMatrix.matvec (problems.py:127-136): elementwise products, then a
    reduceat over every non-empty row segment."""
    x = np.asarray(x, dtype=np.float64)
    products = data * x[indices]
    nrows = len(indptr) - 1
    y = np.zeros(nrows)
    rows = np.flatnonzero(np.diff(indptr) > 0)
    if products.size:
        y[rows] = np.add.reduceat(products, indptr[rows])
    return y


def stencil7_matvec(x, dims):
    """StencilLaplace3D._matvec (problems.py:296-305): 6 g minus the
    neighbours, axis by axis, lower neighbour before upper."""
    g = np.asarray(x, dtype=np.float64).reshape(dims)
    y = 6.0 * g
    full = slice(None)
    for axis in range(3):
        head = [full] * 3
        tail = [full] * 3
        head[axis] = slice(1, None)
        tail[axis] = slice(None, -1)
        y[tuple(head)] -= g[tuple(tail)]  # neighbour at index - 1
        y[tuple(tail)] -= g[tuple(head)]  # neighbour at index + 1
    return y.reshape(-1)


def _coo_to_csr(n, rows, cols, vals):
    """CsrMatrix.from_coo (problems.py:98-117): sort by (row, col), sum
    duplicates in input order."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size == 0:
        return np.zeros(n + 1, dtype=np.int64), cols, vals
    new = np.r_[True, (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])]
    groups = np.cumsum(new) - 1
    acc = np.zeros(int(groups[-1]) + 1)
    np.add.at(acc, groups, vals)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, rows[new] + 1, 1)
    return np.cumsum(indptr), cols[new], acc


def manteuffel_csr(k, beta=0.5):
    """manteuffel_parts + manteuffel_build (problems.py:208-245) with the
    default L = k+1, h = 1: M (5-point, 4/-1) scaled by 1/h^2 plus N
    (centred differences, -1 below / +1 above) scaled by beta/(2h)."""
    h = float(k + 1) / (k + 1)
    diff = 1.0 / (h * h)
    conv = beta / (2.0 * h)
    mr, mc, mv, nr, nc, nv = [], [], [], [], [], []
    for r in range(k * k):
        blk, i = divmod(r, k)
        mr.append(r), mc.append(r), mv.append(4.0)
        for nb, inside, sgn in ((r - 1, i > 0, -1.0), (r - k, blk > 0, -1.0),
                                (r + 1, i < k - 1, 1.0), (r + k, blk < k - 1, 1.0)):
            if inside:
                mr.append(r), mc.append(nb), mv.append(-1.0)
                nr.append(r), nc.append(nb), nv.append(sgn)
    n = k * k
    mp, mi, md = _coo_to_csr(n, mr, mc, mv)
    np_, ni, nd = _coo_to_csr(n, nr, nc, nv)
    rows = np.concatenate([np.repeat(np.arange(n), np.diff(mp)), np.repeat(np.arange(n), np.diff(np_))])
    return _coo_to_csr(n, rows, np.concatenate([mi, ni]), np.concatenate([diff * md, conv * nd]))


def laplace3d_csr(nx, ny, nz):
    """StencilLaplace3D.to_csr (problems.py:307-331)."""
    dims = (nx, ny, nz)
    n = nx * ny * nz
    idx = np.arange(n).reshape(dims)
    rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.full(n, 6.0)]
    for axis in range(3):
        a = np.take(idx, np.arange(dims[axis] - 1), axis=axis).ravel()
        b = np.take(idx, np.arange(1, dims[axis]), axis=axis).ravel()
        rows += [a, b]
        cols += [b, a]
        vals += [np.full(a.size, -1.0)] * 2
    return _coo_to_csr(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def band_random_coo(m, band, d, seed):
    """Config 5's banded random operator (no reference counterpart: the
    generator is this repo's): row i holds d entries, one per
    equal slice of its window [max(0, i-band), min(m, i+band+1)), at column
    slice_lo + (h >> 32) % slice_len with h = mix64(seed * G + i * H + k), value
    (mix64(h ^ C) >> 11) * 2^-53 * 2 - 1.  uint64 arithmetic mod 2^64 -- the
    restatement of csrc/build_ops.cu band_csr_kernel; the reference's
    CsrMatrix.from_coo turns it into the golden CSR."""
    M64 = np.uint64(0xFFFFFFFFFFFFFFFF)

    def mix(x):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))

    i = np.arange(m, dtype=np.int64)
    lo = np.maximum(i - band, 0)
    hi = np.minimum(i + band + 1, m)
    w = hi - lo
    rows, cols, vals = [], [], []
    with np.errstate(over="ignore"):
        for k in range(d):
            a = lo + w * k // d
            b = lo + w * (k + 1) // d
            h = mix(np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
                    + i.astype(np.uint64) * np.uint64(0xD1B54A32D192ED03) + np.uint64(k)) & M64
            c = a + ((h >> np.uint64(32)) % (b - a).astype(np.uint64)).astype(np.int64)
            h2 = mix(h ^ np.uint64(0x5DEECE66D))
            v = (h2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 * 2.0 - 1.0
            rows.append(i)
            cols.append(c)
            vals.append(v)
    # row-major: row i's d entries, ascending columns
    return (np.stack(rows, axis=1).ravel(), np.stack(cols, axis=1).ravel(),
            np.stack(vals, axis=1).ravel())


# ---------------------------------------------------------------------------
# kernels (kernels.py:28-84)


def gram(left, right):
    """mv_trans_mv: left^T right, one reduction (kernels.py:44-60)."""
    return left.T @ right


def _minus_times(y, b, s):
    """mv_times_mat_add_mv(y, b, s, sign=-1) in place (kernels.py:63-84)."""
    if b.shape[1]:
        y += -1.0 * (b @ s)
    return y


def _norm2(x):
    return float(np.sqrt(float(np.dot(x, x))))


# ---------------------------------------------------------------------------
# expansions


class Dcgs2Expansion:
    """_DelayedArnoldi(corrected=True) (arnoldi.py:307-455) as a stepper."""

    def __init__(self, apply, start, capacity, counts=None):
        self.apply = apply
        self.cnt = counts if counts is not None else Counts()
        start = np.asarray(start, dtype=np.float64)
        self.m = m = start.size
        self.cap = capacity
        self.V = np.zeros((m, capacity), order="F")
        self.H = np.zeros((capacity, capacity - 1))
        self.nb = 0
        self.hcols = 0
        self.happy = False
        self.start_norm = None
        self.K = None
        nrm = float(np.linalg.norm(start))
        if not nrm > 0.0:
            raise ValueError("zero start vector")
        self.w = start.copy()
        self.aw = self._A(self.w)
        self.wscale = nrm

    def _A(self, x):
        self.cnt.napply += 1
        return self.apply(x)

    @property
    def order(self):
        size = self.nb + (self.w is not None)
        return size if self.happy else size - 1

    def _complete(self, c, sub):
        j = self.nb
        if j > 0:
            self.H[:j, j - 1] = self.K + c
            self.H[j, j - 1] = sub
            self.hcols = j

    def step(self):
        if self.happy:
            return False
        if self.nb + (self.w is not None) >= self.cap:
            raise IndexError("capacity exhausted")
        m, j, cnt = self.m, self.nb, self.cnt
        Q = self.V[:, :j]
        g = gram(np.hstack([Q, self.w[:, None]]), np.column_stack([self.w, self.aw]))
        cnt.rec("MvTransMv", 2 * m * (j + 1) * 2)
        c, beta, s, s_piv = g[:j, 0], float(g[j, 0]), g[:j, 1], float(g[j, 1])
        if not np.sqrt(max(beta, 0.0)) > EPS * np.sqrt(m) * self.wscale:
            self._complete(c, 0.0)
            self.w = None
            self.happy = True
            return False
        alpha_sq = beta - float(c @ c)
        cnt.flops += 2 * j
        if not alpha_sq > beta * EPS * EPS:
            raise OracleBreakdown("pythagorean", "pythagorean", j)
        alpha = float(np.sqrt(alpha_sq))
        u = self.w[:, None].copy()
        _minus_times(u, Q, c[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        q = u[:, 0] / alpha
        t_piv = (s_piv - float(c @ s)) / (alpha * alpha)
        cnt.flops += 2 * j
        if self.start_norm is None:
            self.start_norm = alpha
        t = np.append(s / alpha, t_piv)
        self._complete(c, alpha)
        self.V[:, j] = q
        self.nb += 1
        hc = self.H[: j + 1, :j] @ c
        cnt.flops += 2 * (j + 1) * j
        self.K = t - hc / alpha
        vscale = float(np.linalg.norm(self.aw)) / alpha
        w = (self.aw / alpha)[:, None]
        cnt.flops += m
        _minus_times(w, self.V[:, : j + 1], t[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * (j + 1))
        self.w = w[:, 0]
        self.aw = self._A(self.w)
        self.wscale = vscale
        return True

    def finalize(self):
        if self.w is not None:
            m, j, cnt = self.m, self.nb, self.cnt
            Q = self.V[:, :j]
            c = gram(Q, self.w[:, None])[:, 0]
            cnt.rec("MvTransMv", 2 * m * j)
            u = self.w[:, None].copy()
            _minus_times(u, Q, c[:, None])
            cnt.rec("MvTimesMatAddMv", 2 * m * j)
            alpha = _norm2(u[:, 0])
            cnt.rec("MvDot", 2 * m)
            self.w = None
            if not alpha > EPS * np.sqrt(m) * self.wscale:
                self._complete(c, 0.0)
                self.happy = True
            else:
                if self.start_norm is None:
                    self.start_norm = alpha
                self._complete(c, alpha)
                self.V[:, j] = u[:, 0] / alpha
                self.nb += 1
        return self.V[:, : self.nb].copy(), self.H[: self.nb, : self.hcols].copy()


class Cgs2Expansion:
    """_ImmediateArnoldi + Cgs2State (arnoldi.py:121-172, ortho.py:139-158)."""

    def __init__(self, apply, start, capacity, counts=None):
        self.apply = apply
        self.cnt = counts if counts is not None else Counts()
        start = np.asarray(start, dtype=np.float64)
        self.m = m = start.size
        self.cap = capacity
        self.V = np.zeros((m, capacity), order="F")
        self.H = np.zeros((capacity, capacity - 1))
        self.hcols = 0
        self.happy = False
        nrm = float(np.linalg.norm(start))
        if not nrm > 0.0:
            raise ValueError("zero start vector")
        self.start_norm = nrm
        self.V[:, 0] = start / nrm
        self.nb = 1

    @property
    def order(self):
        return self.nb if self.happy else self.nb - 1

    def step(self):
        if self.happy:
            return False
        if self.nb >= self.cap:
            raise IndexError("capacity exhausted")
        m, j, cnt = self.m, self.nb, self.cnt
        cnt.napply += 1
        a = self.apply(self.V[:, j - 1])
        scale = float(np.linalg.norm(a))
        Q = self.V[:, :j]
        s = gram(Q, a[:, None])[:, 0]
        cnt.rec("MvTransMv", 2 * m * j)
        w = a.copy()[:, None]
        _minus_times(w, Q, s[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        c = gram(Q, w)[:, 0]
        cnt.rec("MvTransMv", 2 * m * j)
        _minus_times(w, Q, c[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        alpha = _norm2(w[:, 0])
        cnt.rec("MvDot", 2 * m)
        coeffs = s + c
        self.H[:j, j - 1] = coeffs
        self.hcols = j
        if not alpha > EPS * np.sqrt(m) * scale:
            self.H[j, j - 1] = 0.0
            self.happy = True
            return False
        self.H[j, j - 1] = alpha
        self.V[:, j] = w[:, 0] / alpha
        self.nb += 1
        return True

    def finalize(self):
        return self.V[:, : self.nb].copy(), self.H[: self.nb, : self.hcols].copy()


_EXPANSIONS = {"dcgs2": Dcgs2Expansion, "cgs2": Cgs2Expansion}


def _expand(cls, apply, start, steps, counts):
    exp = cls(apply, start, steps + 1, counts)
    while exp.order < steps and exp.step():
        pass
    V, H = exp.finalize()
    return V, H, exp


def dcgs2_arnoldi(apply, start, steps, counts=None):
    """arnoldi_expand(op, start, "dcgs2", steps) (arnoldi.py:603-609)."""
    V, H, exp = _expand(Dcgs2Expansion, apply, start, steps, counts)
    return V, H, exp.cnt


def cgs2_arnoldi(apply, start, steps, counts=None):
    """arnoldi_expand(op, start, "cgs2", steps)."""
    V, H, exp = _expand(Cgs2Expansion, apply, start, steps, counts)
    return V, H, exp.cnt


# ---------------------------------------------------------------------------
# QR (ortho.py)


def cgs2_qr(A, counts=None):
    """qr_factorize(A, "cgs2") (ortho.py:139-158, 492-507)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    cnt = counts if counts is not None else Counts()
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n))
    for j in range(n):
        a = A[:, j]  # strided view, as _take hands the reference's kernels
        scale = float(np.linalg.norm(a))
        Qj = Q[:, :j]
        s = gram(Qj, a[:, None])[:, 0]
        cnt.rec("MvTransMv", 2 * m * j)
        w = a[:, None].copy()
        _minus_times(w, Qj, s[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        c = gram(Qj, w)[:, 0]
        cnt.rec("MvTransMv", 2 * m * j)
        _minus_times(w, Qj, c[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        alpha = _norm2(w[:, 0])
        cnt.rec("MvDot", 2 * m)
        if not alpha > EPS * np.sqrt(m) * scale:
            raise OracleBreakdown("dependent", "dependent", j)
        Q[:, j] = w[:, 0] / alpha
        R[:j, j] = s + c
        R[j, j] = alpha
    return Q, R, cnt


def dcgs2_qr(A, counts=None):
    """qr_factorize(A, "dcgs2") (Dcgs2State, ortho.py:326-413)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    cnt = counts if counts is not None else Counts()
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n))
    nq = 0
    w = s_prev = None
    wscale = 0.0

    def emit(u, coeffs, alpha):
        nonlocal nq
        Q[:, nq] = u / alpha
        R[: len(coeffs), nq] = coeffs
        R[nq, nq] = alpha
        nq += 1

    for col in range(n):
        a = A[:, col]
        if w is None:
            w, s_prev, wscale = a.copy(), np.zeros(0), float(np.linalg.norm(a))
            continue
        j = nq
        Qj = Q[:, :j]
        g = gram(np.hstack([Qj, w[:, None]]), np.column_stack([w, a]))
        cnt.rec("MvTransMv", 2 * m * (j + 1) * 2)
        c, beta, s_new, s_piv = g[:j, 0], float(g[j, 0]), g[:j, 1], float(g[j, 1])
        if not np.sqrt(max(beta, 0.0)) > EPS * np.sqrt(m) * wscale:
            raise OracleBreakdown("dependent", "dependent", j)
        alpha_sq = beta - float(c @ c)
        cnt.flops += 2 * j
        if not alpha_sq > beta * EPS * EPS:
            raise OracleBreakdown("pythagorean", "pythagorean", j)
        alpha = float(np.sqrt(alpha_sq))
        u = w[:, None].copy()
        _minus_times(u, Qj, c[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        emit(u[:, 0], s_prev + c, alpha)
        s_piv = (s_piv - float(c @ s_new)) / alpha
        cnt.flops += 2 * j
        s_full = np.append(s_new, s_piv)
        wn = a.copy()[:, None]
        _minus_times(wn, Q[:, : j + 1], s_full[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * (j + 1))
        w, s_prev, wscale = wn[:, 0], s_full, float(np.linalg.norm(a))
    if w is not None:
        j = nq
        Qj = Q[:, :j]
        c = gram(Qj, w[:, None])[:, 0]
        cnt.rec("MvTransMv", 2 * m * j)
        u = w[:, None].copy()
        _minus_times(u, Qj, c[:, None])
        cnt.rec("MvTimesMatAddMv", 2 * m * j)
        alpha = _norm2(u[:, 0])
        cnt.rec("MvDot", 2 * m)
        if not alpha > EPS * np.sqrt(m) * wscale:
            raise OracleBreakdown("dependent", "dependent", j)
        emit(u[:, 0], s_prev + c, alpha)
    return Q[:, :nq], R[:nq, :nq], cnt


# ---------------------------------------------------------------------------
# GMRES (gmres.py:63-211)


def _givens_append(st, hcol, sub):
    j = st["n"]
    col = np.zeros(j + 2)
    col[: len(hcol)] = hcol
    col[j + 1] = sub
    cs, sn = st["cs"], st["sn"]
    for i in range(j):
        top = cs[i] * col[i] + sn[i] * col[i + 1]
        col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
        col[i] = top
    rad = float(np.hypot(col[j], col[j + 1]))
    cs[j], sn[j] = (1.0, 0.0) if rad == 0.0 else (col[j] / rad, col[j + 1] / rad)
    col[j] = rad
    st["r"][: j + 1, j] = col[: j + 1]
    g = st["g"]
    top = cs[j] * g[j]
    g[j + 1] = -sn[j] * g[j]
    g[j] = top
    st["n"] += 1
    return abs(g[j + 1])


def _givens_solve(st):
    k = st["n"]
    if k == 0:
        return np.zeros(0)
    y = np.zeros(k)
    d = np.abs(np.diag(st["r"][:k, :k]))
    if np.any(d == 0.0):
        k = int(np.argmax(d == 0.0))
        if k == 0:
            return y
    y[:k] = np.linalg.solve(st["r"][:k, :k], st["g"][:k])
    return y


def gmres(apply, b, anorm, max_iters, restart=0, rtol=0.0, scheme="dcgs2"):
    """gmres_solve (gmres.py:115-211) with the reference's per-column
    backward errors; returns a dict of the result fields."""
    cls = _EXPANSIONS[scheme]
    b = np.asarray(b, dtype=np.float64)
    cnt = Counts()
    m = b.size
    x = np.zeros(m)
    bnorm = float(np.linalg.norm(b))
    cycle = restart if restart > 0 else max_iters
    rel, bes, reds = [], [], []
    iters, converged, breakdown, stagnated = 0, False, False, False

    def berr(xj):
        cnt.napply += 1
        r = b - apply(xj)
        den = anorm * float(np.linalg.norm(xj)) + float(np.linalg.norm(b))
        return 0.0 if den == 0.0 else float(np.linalg.norm(r) / den)

    while iters < max_iters and not converged and not breakdown:
        if iters:
            cnt.napply += 1
            r = b - apply(x)
        else:
            r = b.copy()
        budget = min(cycle, max_iters - iters)
        exp = cls(apply, r, budget + 1, cnt)
        st = None
        done = flat = 0
        best = np.inf

        def drain():
            nonlocal st, done, flat, best, stagnated
            while done < exp.hcols:
                if st is None:
                    st = {"n": 0, "r": np.zeros((budget, budget)), "cs": np.zeros(budget),
                          "sn": np.zeros(budget), "g": np.zeros(budget + 1)}
                    st["g"][0] = exp.start_norm
                res = _givens_append(st, exp.H[: done + 1, done], exp.H[done + 1, done]) / bnorm
                rel.append(res)
                y = _givens_solve(st)
                bes.append(berr(x + exp.V[:, : exp.nb][:, : len(y)] @ y))
                reds.append(cnt.reductions)
                if res < best * (1.0 - 1e-12):
                    best, flat = res, 0
                else:
                    flat += 1
                    stagnated = stagnated or flat >= 20
                done += 1

        for _ in range(budget):
            alive = exp.step()
            drain()
            if not alive:
                breakdown = True
                break
            if rtol > 0 and rel and rel[-1] <= rtol:
                break
        V, _ = exp.finalize()
        drain()
        iters += done
        y = _givens_solve(st) if st is not None else np.zeros(0)
        x = x + V[:, : len(y)] @ y
        if rtol > 0 and rel and rel[-1] <= rtol:
            converged = True
        if restart == 0:
            break
    return {"x": x, "residual_history": np.array(rel), "backward_errors": np.array(bes),
            "reduction_history": np.array(reds, dtype=np.int64), "iterations": iters,
            "converged": converged or breakdown, "stagnated": stagnated,
            "breakdown": breakdown, "napply": cnt.napply, "reductions": cnt.reductions}
