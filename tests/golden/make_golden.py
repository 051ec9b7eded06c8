"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports kls 0.1.0 from /root/reference/pkg/src, runs the hot-path entry
points on small seeded inputs, and stores inputs and outputs as compressed
npz files.  The GPU box never runs this script; the tests only read the
committed fixtures.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def ledger_fields(led):
    return dict(reductions=led.reductions, flops=led.flops,
                mvtransmv=led.kernel_counts["MvTransMv"],
                mvtimes=led.kernel_counts["MvTimesMatAddMv"], mvdot=led.kernel_counts["MvDot"])


def main():
    sys.path.insert(0, REF)
    import kls
    from kls.ortho import Dcgs2State

    rng = np.random.Generator(np.random.PCG64(20240915))

    # -- CSR matvec with ragged rows (pairwise summation branches) ----------
    lengths = [0, 1, 2, 3, 7, 8, 9, 15, 16, 17, 64, 127, 128, 129, 130, 200, 256, 257, 300, 0, 5]
    n = 400
    rows, cols, vals = [], [], []
    for r, L in enumerate(lengths):
        c = np.sort(rng.choice(n, size=L, replace=False))
        rows += [r] * L
        cols += list(c)
        vals += list(rng.standard_normal(L) * 10.0 ** rng.integers(-6, 7, size=L))
    csr = kls.CsrMatrix.from_coo(len(lengths), n, rows, cols, vals)
    x = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, size=n)
    np.savez_compressed(os.path.join(OUT, "csr_ragged.npz"), indptr=csr.indptr,
                        indices=csr.indices, data=csr.data, x=x, y=csr.matvec(x))

    # -- stencil and generators ----------------------------------------------
    out = {}
    for dims in ((5, 4, 6), (1, 1, 1), (3, 1, 7), (8, 8, 8)):
        op = kls.laplace3d(*dims)
        xs = rng.standard_normal(op.n)
        key = "x".join(map(str, dims))
        out[f"x_{key}"] = xs
        out[f"y_{key}"] = op.apply(xs)
        out[f"fro_{key}"] = op.frobenius_norm()
        c = op.to_csr()
        out[f"csr_indptr_{key}"], out[f"csr_indices_{key}"], out[f"csr_data_{key}"] = (
            c.indptr, c.indices, c.data)
    for k, beta in ((1, 0.5), (2, 0.5), (4, 0.5), (7, 0.3), (10, 0.5), (6, 0.0)):
        a = kls.manteuffel_build(kls.ManteuffelSpec(k=k, beta=beta))
        out[f"mant_indptr_{k}_{beta}"] = a.indptr
        out[f"mant_indices_{k}_{beta}"] = a.indices
        out[f"mant_data_{k}_{beta}"] = a.data
        out[f"mant_eigs_{k}_{beta}"] = kls.manteuffel_eigenvalues(
            kls.ManteuffelSpec(k=k, beta=beta)).values
    np.savez_compressed(os.path.join(OUT, "operators.npz"), **out)

    # -- Arnoldi: Manteuffel k=10 (tests/test_arnoldi.py fixtures) -----------
    out = {}
    op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=10)))
    start = np.random.Generator(np.random.PCG64(77)).standard_normal(100)
    out["start"] = start
    for scheme in ("dcgs2", "cgs2"):
        led = kls.SyncLedger()
        op.napply = 0
        V, H = kls.arnoldi_expand(op, start, scheme, steps=40, ledger=led)
        out[f"{scheme}_V"], out[f"{scheme}_H"] = V, H
        out[f"{scheme}_napply"] = op.napply
        for kk, vv in ledger_fields(led).items():
            out[f"{scheme}_{kk}"] = vv
    # per-step reduction counts and a mid-run snapshot
    exp = kls.arnoldi(op, start, "dcgs2", capacity=10)
    for _ in range(6):
        exp.step()
    out["mid_h_ext"] = exp.h_extended.copy()
    out["mid_basis_ext"] = exp.basis_extended.copy()
    # resume from a cgs2 decomposition with a dense coupling row
    v0, h0 = kls.arnoldi_expand(op, start, "cgs2", steps=8)
    hbar = h0.copy()
    hbar[8, :] = 0.3 * np.arange(1.0, 9.0)
    out["resume_v0"], out["resume_hbar"] = v0, hbar
    for scheme in ("dcgs2", "cgs2"):
        led = kls.SyncLedger()
        e = kls.resume_arnoldi(op, v0, hbar, scheme, capacity=20, ledger=led)
        while e.order < 14:
            e.step()
        V, H = e.finalize()
        out[f"resume_{scheme}_V"], out[f"resume_{scheme}_H"] = V, H
        out[f"resume_{scheme}_reductions"] = led.reductions
    np.savez_compressed(os.path.join(OUT, "arnoldi_m10.npz"), **out)

    # -- config 1: 2D Poisson 100x100 (beta = 0), n = 50, dcgs2 and cgs2 ------
    out = {}
    op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
    for scheme in ("dcgs2", "cgs2"):
        led = kls.SyncLedger()
        V, H = kls.arnoldi_expand(op, start, scheme, steps=50, ledger=led)
        out[f"{scheme}_H"] = H
        out[f"{scheme}_Vsub"] = V[::97]
        out[f"{scheme}_Vcolsum"] = V.sum(axis=0)
        out[f"{scheme}_loo"] = kls.loss_of_orthogonality(V)
        out[f"{scheme}_rre"] = kls.representation_error_arnoldi(op, V, H)
        out[f"{scheme}_reductions"] = led.reductions
    np.savez_compressed(os.path.join(OUT, "arnoldi_poisson100.npz"), **out)

    # -- matrix-free 3-D Laplacian, dcgs2 / cgs2 --------------------------------
    out = {}
    op = kls.laplace3d(6, 5, 4)
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
    out["start"] = start
    for scheme in ("dcgs2", "cgs2"):
        V, H = kls.arnoldi_expand(op, start, scheme, steps=30)
        out[f"{scheme}_V"], out[f"{scheme}_H"] = V, H
    np.savez_compressed(os.path.join(OUT, "arnoldi_laplace3d.npz"), **out)

    # -- QR --------------------------------------------------------------------
    out = {}
    a = rng.standard_normal((100, 10))
    out["A"] = a
    for scheme in ("dcgs2", "cgs2"):
        led = kls.SyncLedger()
        q, r = kls.qr_factorize(a, scheme, ledger=led)
        out[f"{scheme}_Q"], out[f"{scheme}_R"] = q, r
        for kk, vv in ledger_fields(led).items():
            out[f"{scheme}_{kk}"] = vv
    ak = kls.synthetic_kappa(100, 10, 1e4, seed=17)
    out["Akappa"] = ak
    for scheme in ("dcgs2", "cgs2"):
        q, r = kls.qr_factorize(ak, scheme)
        out[f"kappa_{scheme}_Q"], out[f"kappa_{scheme}_R"] = q, r
    st = Dcgs2State(3, 3)
    st._q[:, 0] = [0.0, 0.0, 1.0]
    st.ncols = 1
    st.npushed = 1
    st._w = np.array([3.0, 4.0, 1.0])
    st._s = np.array([0.0])
    st._wscale = float(np.linalg.norm(st._w))
    st.npushed += 1
    st.push(np.array([1.0, 0.0, 0.0]))
    out["hand_R"] = st._r.copy()
    out["hand_Q"] = st._q.copy()
    np.savez_compressed(os.path.join(OUT, "qr.npz"), **out)

    # -- GMRES -------------------------------------------------------------------
    out = {}
    cases = {
        "mant12": (kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=12))), 10, 1e-8, 400),
        "lap8": (kls.laplace3d(8, 8, 8), 0, 0.0, 60),
        "mant100": (kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100))), 50, 1e-6,
                    10000),
    }
    for name, (op, restart, rtol, iters) in cases.items():
        one = op.apply(np.ones(op.n))
        b = one / np.linalg.norm(one)
        out[f"{name}_b"] = b
        for scheme in ("dcgs2", "cgs2"):
            if name == "mant100" and scheme == "cgs2":
                continue
            led = kls.SyncLedger()
            res = kls.gmres_solve(op, b, kls.GmresConfig(max_iters=iters, restart=restart,
                                                         rtol=rtol, scheme=scheme), ledger=led)
            p = f"{name}_{scheme}"
            out[f"{p}_iterations"] = res.iterations
            out[f"{p}_residual_history"] = res.residual_history
            out[f"{p}_backward_errors"] = res.backward_errors
            out[f"{p}_reduction_history"] = res.reduction_history
            out[f"{p}_converged"] = res.converged
            out[f"{p}_x"] = res.x if op.n <= 1000 else res.x[::97]
    np.savez_compressed(os.path.join(OUT, "gmres.npz"), **out)

    # -- Krylov-Schur ------------------------------------------------------------
    out = {}
    for name, k, mb, seed, rst, scheme in (("k5", 5, 25, 3, 100, "dcgs2"),
                                           ("k8", 8, 30, 11, 8, "dcgs2"),
                                           ("k10", 10, 20, 5, 30, "dcgs2"),
                                           ("k10c", 10, 20, 5, 30, "cgs2")):
        spec = kls.ManteuffelSpec(k=k)
        op = kls.CsrOperator(kls.manteuffel_build(spec))
        cfg = kls.KrylovSchurConfig(max_basis=mb, tol=1e-7, scheme=scheme, max_restarts=rst)
        res = kls.krylov_schur_run(op, cfg, seed=seed, exact=kls.manteuffel_eigenvalues(spec))
        out[f"{name}_values"] = res.values
        out[f"{name}_residuals"] = res.residuals
        out[f"{name}_lock_history"] = np.array(res.lock_history)
        out[f"{name}_restarts"] = res.restarts
        out[f"{name}_invariant_dim"] = res.invariant_dim
        out[f"{name}_incomplete"] = res.incomplete
        out[f"{name}_over"] = res.over_multiplicity
        # the reference's own sensitivity: the same matrix applied as a
        # DenseOperator (only the matvec summation order changes)
        alt = kls.krylov_schur_run(kls.DenseOperator(op.to_dense()), cfg, seed=seed)
        out[f"{name}_alt_lock_history"] = np.array(alt.lock_history)
        out[f"{name}_alt_values"] = alt.values
    np.savez_compressed(os.path.join(OUT, "krylov_schur.npz"), **out)

    # -- small dense Schur services (host side of Krylov-Schur) ------------------
    from kls.schur import (SchurForm, hessenberg_real_schur, hessenberg_reduce,
                           move_blocks_front, schur_eigenvectors, sort_schur)
    out = {}
    srng = np.random.Generator(np.random.PCG64(4242))
    for i, n in enumerate((1, 2, 3, 5, 8, 13, 21, 30, 30, 45)):
        a = srng.standard_normal((n, n))
        if i == 8:  # clustered real spectrum plus a rotation block
            q = np.linalg.qr(srng.standard_normal((n, n)))[0]
            d = np.diag(np.repeat(np.arange(1.0, 11.0), 3))
            d[0, 1], d[1, 0] = 0.5, -0.5
            a = q @ d @ q.T
        h, u = hessenberg_reduce(a)
        f = hessenberg_real_schur(h)
        sel = srng.random(len(f.blocks())) < 0.4
        g = SchurForm(f.t.copy(), f.z.copy())
        moved = move_blocks_front(g, sel)
        vals, vecs = schur_eigenvectors(g)
        srt = SchurForm(f.t.copy(), f.z.copy())
        sort_schur(srt, lambda lam: lam.real)
        out[f"a{i}"], out[f"h{i}"], out[f"u{i}"] = a, h, u
        out[f"t{i}"], out[f"z{i}"] = f.t, f.z
        out[f"sel{i}"], out[f"moved{i}"] = sel, moved
        out[f"mt{i}"], out[f"mz{i}"] = g.t, g.z
        out[f"vals{i}"], out[f"vecs{i}"] = vals, vecs
        out[f"st{i}"], out[f"sz{i}"] = srt.t, srt.z
    np.savez_compressed(os.path.join(OUT, "schur.npz"), **out)

    # -- kls-bench CLI outputs (data rows) and the QR-sweep generator ----------
    import contextlib
    import io
    from kls import cli

    out = {}
    runs = {
        "sync": ["sync-count", "--rows", "600", "--cols", "20"],
        "qr": ["qr-stability", "--rows", "120", "--cols", "12", "--kappa-list", "1e0,1e4,1e8"],
        "arnoldi": ["arnoldi-stability", "--manteuffel-k", "12", "--steps", "30", "--stride", "10"],
        "gmres": ["gmres", "--laplace-dims", "6,5,4", "--steps", "25", "--restart", "10"],
        "eig": ["eig", "--manteuffel-k", "6", "--restart-list", "12,20", "--max-restarts", "10"],
    }
    for name, argv in runs.items():
        argv = argv + ["--scheme", "dcgs2", "--scheme", "cgs2"]
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            rc = cli.main(argv)
        out[f"{name}_argv"] = np.array(argv)
        out[f"{name}_rc"] = rc
        out[f"{name}_csv"] = np.array(buf.getvalue())
    out["kappa_matrix"] = kls.synthetic_kappa(60, 8, 1e6, seed=3)
    np.savez_compressed(os.path.join(OUT, "cli.npz"), **out)

    mtx_corpus(kls)
    print("golden fixtures written to", OUT)


def mtx_corpus(kls):
    """The reference's Matrix Market corpus (pkg/tests/data/*.mtx) with its
    parse results, for the host-side parser tests -> mtx_corpus.json."""
    import glob
    import json

    data = os.path.join(os.path.dirname(REF), "tests", "data")
    corpus = {}
    for path in sorted(glob.glob(os.path.join(data, "*.mtx"))):
        entry = {"text": open(path).read()}
        try:
            csr = kls.parse_matrix_market(path)
            entry.update(ok=True, nrows=int(csr.nrows), ncols=int(csr.ncols),
                         indptr=csr.indptr.tolist(), indices=csr.indices.tolist(),
                         data=csr.data.tolist())
        except kls.MatrixMarketError as err:
            entry.update(ok=False, line=err.line)
        corpus[os.path.basename(path)] = entry
    with open(os.path.join(OUT, "mtx_corpus.json"), "w") as f:
        json.dump(corpus, f, indent=1, sort_keys=True)


def gmres_config2(kls):
    """BASELINE config 2 at full size: GMRES(50) with DCGS2 on the 1000 x 1000
    convection-diffusion operator (ManteuffelSpec(k=1000, beta=0.5), m = 1e6),
    b = A 1 / ||A 1|| (cli.py:255-257), rtol 1e-6.  ~12 min of reference CPU
    time; stores the iteration count, the residual history and the
    cumulative reduction history (small) for the iteration-parity test."""
    import time

    op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=1000, beta=0.5)))
    one = op.apply(np.ones(op.n))
    b = one / np.linalg.norm(one)
    led = kls.SyncLedger()
    t0 = time.perf_counter()
    res = kls.gmres_solve(op, b, kls.GmresConfig(max_iters=10000, restart=50, rtol=1e-6,
                                                 scheme="dcgs2"), ledger=led)
    out = {"iterations": res.iterations, "converged": res.converged,
           "residual_history": res.residual_history,
           "backward_errors": res.backward_errors,
           "reduction_history": res.reduction_history,
           "reductions": led.reductions, "cpu_s": time.perf_counter() - t0,
           "x_sample": res.x[::997]}
    # the reference's own noise floor: the same solve under another BLAS
    # thread count (a different summation order in OpenBLAS's dot / gemv).
    # Run the script with OPENBLAS_NUM_THREADS=1; this second solve uses 8.
    from threadpoolctl import threadpool_limits

    with threadpool_limits(limits=8, user_api="blas"):
        res8 = kls.gmres_solve(op, b, kls.GmresConfig(max_iters=10000, restart=50, rtol=1e-6,
                                                      scheme="dcgs2"))
    out["iterations_threads8"] = res8.iterations
    out["residual_history_threads8"] = res8.residual_history
    np.savez_compressed(os.path.join(OUT, "gmres_config2.npz"), **out)


def ks_config4_shape(kls):
    """BASELINE config 4's Krylov-Schur settings (nonsymmetric convection-
    diffusion beta = 0.5, max_basis 60, tol 1e-7, DCGS2, seed 1729) at
    k = 100 (m = 1e4), 30 restarts: the reference's run (run the script with
    OPENBLAS_NUM_THREADS=1) and, for its own sensitivity, the same run under
    8 BLAS threads (a different summation order in OpenBLAS's dot / gemv)."""
    from threadpoolctl import threadpool_limits

    spec = kls.ManteuffelSpec(k=100, beta=0.5)
    op = kls.CsrOperator(kls.manteuffel_build(spec))
    cfg = kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=30)
    out = {}
    for tag, nthr in (("", 1), ("alt_", 8)):
        with threadpool_limits(limits=nthr, user_api="blas"):
            res = kls.krylov_schur_run(op, cfg, seed=1729)
        out[f"{tag}values"] = res.values
        out[f"{tag}lock_history"] = np.array(res.lock_history)
        out[f"{tag}restarts"] = res.restarts
        out[f"{tag}invariant_dim"] = res.invariant_dim
        out[f"{tag}incomplete"] = res.incomplete
    np.savez_compressed(os.path.join(OUT, "ks_config4_shape.npz"), **out)


def ks_config4_full(kls, max_restarts=240):
    """BASELINE config 4 at FULL size: Krylov-Schur on ManteuffelSpec(k=3163,
    beta=0.5) (m = 10,004,569), max_basis 60, tol 1e-7, DCGS2, seed 1729
    (eig.py:157-317).  Hours of reference CPU time, so the run is
    instrumented rather than repeated: every restart's active Hessenberg
    block (the input of eig._schur_active) is captured, and a checkpoint
    (`ks_config4_full.npz`) is rewritten after every restart -- the Ritz
    values of each restart, the active block size (nlock = k - na), and the
    blocks themselves for the first 12 restarts.  When the run ends the
    locked values, lock history and restart count are added.  Threads: the
    OpenBLAS default of the process (recorded)."""
    import time

    from threadpoolctl import threadpool_info

    import kls.eig as keig

    path = os.path.join(OUT, "ks_config4_full.npz")
    rec = {"ritz": [], "na": [], "blocks": [], "t": []}
    t0 = time.perf_counter()
    nthreads = max([d.get("num_threads", 0) for d in threadpool_info()
                    if d.get("user_api") == "blas"] or [0])
    orig = keig._schur_active

    def save(extra=None):
        na = np.array(rec["na"], dtype=np.int64)
        ritz = np.zeros((len(na), 60), dtype=np.complex128)
        for i, v in enumerate(rec["ritz"]):
            ritz[i, : v.size] = v
        out = dict(ritz=ritz, na=na, restart_s=np.array(rec["t"]), blas_threads=nthreads,
                   k=3163, beta=0.5, max_basis=60, tol=1e-7, seed=1729)
        for i, b in enumerate(rec["blocks"]):
            out[f"block{i}"] = b
        if extra:
            out.update(extra)
        tmp = path + ".tmp.npz"
        np.savez_compressed(tmp, **out)
        os.replace(tmp, path)

    def spy(block):
        rec["na"].append(block.shape[0])
        rec["ritz"].append(np.sort_complex(np.linalg.eigvals(block)))
        if len(rec["blocks"]) < 12:
            rec["blocks"].append(block.copy())
        rec["t"].append(time.perf_counter() - t0)
        save()
        print(f"restart {len(rec['na'])}: na={block.shape[0]} t={rec['t'][-1]:.0f}s", flush=True)
        return orig(block)

    keig._schur_active = spy
    op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=3163, beta=0.5)))
    cfg = kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=max_restarts)
    res = keig.krylov_schur_run(op, cfg, seed=1729)
    save(dict(values=res.values, lock_history=np.array(res.lock_history), restarts=res.restarts,
              invariant_dim=res.invariant_dim, incomplete=res.incomplete, done=True,
              cpu_s=time.perf_counter() - t0))


def ks_config4_ensemble(kls, nperm=24):
    """The reference's OWN rounding sensitivity at BASELINE config 4's
    Krylov-Schur settings (k = 100, m = 1e4, max_basis 60, tol 1e-7, DCGS2,
    seed 1729, 30 restarts): the same problem run under exact symmetric row
    permutations P A P^T with the permuted start vector (identical spectrum
    and Krylov spaces in exact arithmetic; only the summation order of the
    dot products / gemvs changes) and under 1, 2, 4, 8 BLAS threads.  The
    lock histories and locked values of these runs are the envelope a
    re-implementation with a different summation order must fall into
    (SURVEY.md section 8c).  Stored: lock histories (runs x 30), locked
    values (runs x 60, zero-padded, sorted), locked counts."""
    import scipy.sparse as sp
    from threadpoolctl import threadpool_limits

    import kls.eig as keig

    csr = kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.5))
    m = csr.nrows
    cfg = kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=30)
    S = sp.csr_matrix((csr.data, csr.indices, csr.indptr), shape=(m, m))
    real_np = keig.np

    class PermGen:
        def __init__(self, bitgen, perm):
            self.g = real_np.random.Generator(bitgen)
            self.perm = perm

        def standard_normal(self, size=None):
            x = self.g.standard_normal(size)
            return x[self.perm] if np.ndim(x) == 1 and len(x) == len(self.perm) else x

        def __getattr__(self, k):
            return getattr(self.g, k)

    runs = []
    for tag, perm, nthr in ([(f"threads{t}", None, t) for t in (1, 2, 4, 8)] +
                            [(f"perm{t}", np.random.default_rng(100 + t).permutation(m), 1)
                             for t in range(nperm)]):
        if perm is None:
            op = kls.CsrOperator(csr)
            keig.np = real_np
        else:
            Sp = S[perm][:, perm].tocsr()
            Sp.sort_indices()
            op = kls.CsrOperator(kls.CsrMatrix(m, m, Sp.indptr.astype(np.int64),
                                               Sp.indices.astype(np.int64), Sp.data.copy()))
            wrap = type(sys)("np_perm")
            wrap.__dict__.update(real_np.__dict__)
            wrap.random = type(sys)("np_perm_random")
            wrap.random.__dict__.update(real_np.random.__dict__)
            wrap.random.Generator = lambda bg, perm=perm: PermGen(bg, perm)
            keig.np = wrap
        try:
            with threadpool_limits(limits=nthr, user_api="blas"):
                res = keig.krylov_schur_run(op, cfg, seed=1729)
        finally:
            keig.np = real_np
        vals = np.zeros(60, dtype=np.complex128)
        v = np.sort_complex(res.values)
        vals[: v.size] = v
        runs.append((tag, np.array(res.lock_history), vals, v.size))
        print(tag, [(i, int(x)) for i, x in enumerate(res.lock_history)
                    if i == 0 or res.lock_history[i] != res.lock_history[i - 1]], flush=True)
    np.savez_compressed(os.path.join(OUT, "ks_config4_ensemble.npz"),
                        tags=np.array([r[0] for r in runs]),
                        lock_history=np.stack([r[1] for r in runs]),
                        values=np.stack([r[2] for r in runs]),
                        nlocked=np.array([r[3] for r in runs]))


def band_random(kls):
    """Config 5's Arnoldi variant: the banded random operator of
    oracle.band_random_coo assembled by the reference's CsrMatrix.from_coo
    (problems.py:99-117) -- golden CSR arrays for several shapes, edge and
    interior rows -- and the reference's DCGS2 / CGS2 Arnoldi on it at
    m = 50,000 (band 1000, 7 per row), 60 steps, start PCG64(1729)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    import oracle

    out = {}
    for tag, (m, band, d, seed) in {"small": (37, 4, 3, 11), "edge": (1000, 999, 8, 5),
                                    "mid": (50_000, 1000, 7, 2525)}.items():
        r, c, v = oracle.band_random_coo(m, band, d, seed)
        csr = kls.CsrMatrix.from_coo(m, m, r, c, v)
        out[f"{tag}_shape"] = np.array([m, band, d, seed])
        keep = slice(None) if m <= 1000 else np.r_[0:7000, csr.nnz - 7000:csr.nnz]
        out[f"{tag}_indptr"] = csr.indptr if m <= 1000 else csr.indptr[::97]
        out[f"{tag}_indices"], out[f"{tag}_data"] = csr.indices[keep], csr.data[keep]
        out[f"{tag}_datasum"] = np.array([np.sum(csr.data), np.sum(csr.indices)])
    m, band, d, seed = 50_000, 1000, 7, 2525
    r, c, v = oracle.band_random_coo(m, band, d, seed)
    op = kls.CsrOperator(kls.CsrMatrix.from_coo(m, m, r, c, v))
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(m)
    for scheme in ("dcgs2", "cgs2"):
        led = kls.SyncLedger()
        V, H = kls.arnoldi_expand(op, start, scheme, steps=60, ledger=led)
        out[f"arnoldi_{scheme}_H"] = H
        out[f"arnoldi_{scheme}_Vrows"] = V[::997]
        out[f"arnoldi_{scheme}_reductions"] = led.reductions
    np.savez_compressed(os.path.join(OUT, "band_random.npz"), **out)


def arnoldi_config3_shape(kls):
    """BASELINE config 3's expansion (3-D Poisson 7-point, x slowest, n = 100,
    start PCG64(1729)) on one GPU's share of the 8-GPU split scaled down:
    laplace3d(62, 64, 64), m = 253,952.  DCGS2 and CGS2; H, loss of
    orthogonality, ledger counts, a row sample of V; plus the DCGS2 H under
    8 BLAS threads (the reference's own summation-order spread)."""
    from threadpoolctl import threadpool_limits

    op = kls.laplace3d(62, 64, 64)
    m = op.shape[0]
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(m)
    out = {}
    for scheme, nthr, tag in (("dcgs2", 1, "dcgs2"), ("cgs2", 1, "cgs2"), ("dcgs2", 8, "dcgs2_t8")):
        op.napply = 0
        with threadpool_limits(limits=nthr, user_api="blas"):
            led = kls.SyncLedger()
            exp = kls.arnoldi(op, start, scheme, 101, ledger=led)
            for _ in range(100):
                exp.step()
            V, H = exp.finalize()
        out[f"{tag}_H"] = H
        if nthr == 1:
            G = V.T @ V
            out[f"{tag}_loo"] = np.linalg.norm(np.eye(G.shape[0]) - G)
            out[f"{tag}_Vrows"] = V[::4999]
            for k, v in ledger_fields(led).items():
                out[f"{tag}_{k}"] = v
            out[f"{tag}_napply"] = op.napply
    np.savez_compressed(os.path.join(OUT, "arnoldi_config3_shape.npz"), **out)


def _config5_matrix(m, n, seed=2525, density=1e-3):
    """Config 5's random-sparse tall-skinny shape: each column has
    round(density * m) N(0, 1) entries at distinct random rows."""
    rng = np.random.Generator(np.random.PCG64(seed))
    A = np.zeros((m, n))
    nnz = max(1, int(round(density * m)))
    for c in range(n):
        rows = rng.choice(m, size=nnz, replace=False)
        A[rows, c] = rng.standard_normal(nnz)
    return A


def qr_config5_shape(kls):
    """DCGS2 / CGS2 QR of config 5's matrix shape at m = 250,000, n = 100
    (density 1e-3): R, loss of orthogonality, ledger counts and a row sample
    of Q from the reference; the matrix is regenerated by the test from the
    same seed (_config5_matrix, copied there)."""
    from threadpoolctl import threadpool_limits

    A = _config5_matrix(250_000, 100)
    out = {}
    for scheme, nthr, tag in (("dcgs2", 1, "dcgs2"), ("cgs2", 1, "cgs2"), ("dcgs2", 8, "dcgs2_t8")):
        with threadpool_limits(limits=nthr, user_api="blas"):
            led = kls.SyncLedger()
            Q, R = kls.qr_factorize(A, scheme, ledger=led)
        out[f"{tag}_R"] = R
        if nthr == 1:
            out[f"{tag}_loo"] = np.linalg.norm(np.eye(Q.shape[1]) - Q.T @ Q)
            out[f"{tag}_Qrows"] = Q[::4999]
            for k, v in ledger_fields(led).items():
                out[f"{tag}_{k}"] = v
    out["Asum"] = A.sum(axis=0)
    np.savez_compressed(os.path.join(OUT, "qr_config5_shape.npz"), **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["--only", "mtx"]:
        sys.path.insert(0, REF)
        import kls

        mtx_corpus(kls)
    elif sys.argv[1:] == ["--only", "arnoldi_config3_shape"]:
        sys.path.insert(0, REF)
        import kls

        arnoldi_config3_shape(kls)
    elif sys.argv[1:] == ["--only", "qr_config5_shape"]:
        sys.path.insert(0, REF)
        import kls

        qr_config5_shape(kls)
    elif sys.argv[1:] == ["--only", "ks_config4_shape"]:
        sys.path.insert(0, REF)
        import kls

        ks_config4_shape(kls)
    elif sys.argv[1:2] == ["--only"] and sys.argv[2:3] == ["ks_config4_full"]:
        sys.path.insert(0, REF)
        import kls

        ks_config4_full(kls, *(int(a) for a in sys.argv[3:4]))
    elif sys.argv[1:] == ["--only", "ks_config4_ensemble"]:
        sys.path.insert(0, REF)
        import kls

        ks_config4_ensemble(kls)
    elif sys.argv[1:] == ["--only", "band_random"]:
        sys.path.insert(0, REF)
        import kls

        band_random(kls)
    elif sys.argv[1:] == ["--only", "gmres_config2"]:
        sys.path.insert(0, REF)
        import kls

        gmres_config2(kls)
    else:
        main()
