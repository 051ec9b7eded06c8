"""``kls-bench`` on the B200 backend (reference cli.py): the same
subcommands, CSV schema, ``#`` provenance headers and exit codes, running
every solve on the GPU.

    python -m paper_2104_01253_b200.cli <subcommand> [options]

Subcommands: qr-stability, arnoldi-stability, eig, gmres, sync-count,
mm-run.  Schemes: dcgs2 and cgs2 (the north-star pair); other reference ids
exit with code 2.  Exit codes: 0 success, 2 configuration error, 3 assertion
failure (sync-count mismatch, eigenvalue over-multiplicity), 4 a numerical
breakdown halted a run.  ``--jobs`` is accepted for compatibility; sweep
points run one after another on the device (deterministic order).
"""

import argparse
import os
import sys

import numpy as np

from . import __version__
from .arnoldi import arnoldi
from .eig import KrylovSchurConfig, krylov_schur_run, match_eigenvalues
from .errors import BreakdownError, DimensionError, MatrixMarketError
from .gmres import GmresConfig, gmres_solve
from .ledger import SyncLedger, assert_matches, predicted_counts
from .metrics import (StabilityReport, loss_of_orthogonality, representation_error_arnoldi,
                      representation_error_qr)
from .ortho import SCHEME_IDS, qr_factorize
from .problems import (CsrOperator, ManteuffelSpec, laplace3d, manteuffel_build,
                       manteuffel_eigenvalues, parse_matrix_market)

DEFAULT_SEED = 1729
SEED_ENV = "KLS_DEFAULT_SEED"


class _ConfigError(Exception):
    pass


def _floats(text, cast=float):
    try:
        return [cast(t) for t in text.split(",") if t.strip()]
    except ValueError:
        raise _ConfigError(f"bad list {text!r}") from None


def _seed(args):
    if args.seed is not None:
        return args.seed
    env = os.environ.get(SEED_ENV)
    if env is None:
        return DEFAULT_SEED
    try:
        return int(env)
    except ValueError:
        raise _ConfigError(f"bad {SEED_ENV}={env!r}") from None


def _schemes(args, default):
    chosen = args.scheme or list(default)
    for s in chosen:
        if s not in SCHEME_IDS:
            raise _ConfigError(f"scheme {s!r} is not provided by the B200 backend "
                               f"({', '.join(SCHEME_IDS)})")
    return chosen


def _fmt(x):
    return f"{x:.17e}" if isinstance(x, float) else str(x)


def _write(args, header, columns, rows):
    text = [f"# kls-bench {__version__} (b200)", f"# subcommand: {args.command}"]
    text += [f"# {k}: {v}" for k, v in header]
    text.append(columns)
    text.extend(rows)
    blob = "\n".join(text) + "\n"
    if args.out:
        with open(args.out, "w", encoding="ascii") as f:
            f.write(blob)
    else:
        sys.stdout.write(blob)


# ---------------------------------------------------------------------------
# host data generators of the stability studies (dense.py:88-127,
# problems.py:347-361), restated so the sweeps see the reference's matrices


def _householder_thin_q(a):
    a = np.array(a, dtype=np.float64, order="F")
    m, n = a.shape
    refl = np.zeros((m, n))
    betas = np.zeros(n)
    for j in range(n):
        x = a[j:, j]
        tail = float(np.dot(x[1:], x[1:]))
        v = x.copy()
        v[0] = 1.0
        if tail == 0.0:
            beta = 0.0 if x[0] >= 0.0 else 2.0
        else:
            mu = np.sqrt(x[0] * x[0] + tail)
            head = x[0] - mu if x[0] <= 0.0 else -tail / (x[0] + mu)
            beta = 2.0 * head * head / (tail + head * head)
            v[1:] = x[1:] / head
        refl[j:, j] = v
        betas[j] = beta
        if beta != 0.0:
            blk = a[j:, j:]
            w = blk.T @ v[:, None]
            blk += -1.0 * (v[:, None] @ (beta * w).T)
            a[j + 1 :, j] = 0.0
    q = np.eye(m, n)
    for j in range(n - 1, -1, -1):
        if betas[j] == 0.0:
            continue
        v = refl[j:, j]
        w = betas[j] * (v @ q[j:, :])
        q[j:, :] -= np.outer(v, w)
    return q


def synthetic_kappa(m, n, kappa, seed):
    """U diag(sigma) V^T with log-spaced sigma from 1 to 1/kappa."""
    if kappa < 1.0:
        raise ValueError("kappa >= 1 required")
    u = _householder_thin_q(np.random.Generator(np.random.PCG64(seed)).standard_normal((m, n)))
    v = _householder_thin_q(np.random.Generator(np.random.PCG64(seed + 1)).standard_normal((n, n)))
    sigma = np.ones(n) if kappa == 1.0 else np.logspace(0.0, -np.log10(kappa), n)
    return (u * sigma) @ v.T


# ---------------------------------------------------------------------------
# subcommands


def _operator(args):
    if args.mtx:
        csr = parse_matrix_market(args.mtx)
        if csr.nrows != csr.ncols:
            raise _ConfigError("matrix must be square")
        return CsrOperator(csr), f"mtx:{args.mtx}"
    spec = ManteuffelSpec(k=args.manteuffel_k, beta=args.beta)
    return CsrOperator(manteuffel_build(spec)), f"manteuffel:k={spec.k},beta={spec.beta}"


def _cmd_qr_stability(args):
    seed = _seed(args)
    kappas = _floats(args.kappa_list)
    schemes = _schemes(args, SCHEME_IDS)
    rows = []
    for scheme in schemes:
        for kappa in kappas:
            a = synthetic_kappa(args.rows, args.cols, kappa, seed)
            led = SyncLedger()
            try:
                q, r = qr_factorize(a, scheme, ledger=led)
                rep = StabilityReport(scheme=scheme, step=args.cols, loo=loss_of_orthogonality(q),
                                      rre=representation_error_qr(a, q, r), kappa=kappa)
                loo, rre, status = rep.loo, rep.rre, "ok"
            except BreakdownError as err:
                loo = rre = float("nan")
                status = f"breakdown-{err.kind}"
            rows.append(",".join([scheme, _fmt(kappa), str(args.rows), str(args.cols), _fmt(loo),
                                  _fmt(rre), str(led.reductions), status]))
    _write(args, [("schemes", "|".join(schemes)), ("kappas", args.kappa_list),
                  ("rows", args.rows), ("cols", args.cols), ("seed", seed)],
           "scheme,kappa,m,n,loo,rre,reductions,status", rows)
    return 0


def _stability_rows(op, start, scheme, steps, stride, tail):
    led = SyncLedger()
    out = []
    exp = arnoldi(op, start, scheme, capacity=steps + 1, ledger=led)
    try:
        for step in range(1, steps + 1):
            alive = exp.step()
            if step % stride == 0 or not alive or step == steps:
                rep = StabilityReport(scheme=scheme, step=step,
                                      loo=loss_of_orthogonality(exp.basis),
                                      rre=representation_error_arnoldi(
                                          op, exp.basis_extended, exp.h_extended))
                out.append(",".join([scheme, str(step), _fmt(rep.loo), _fmt(rep.rre)]
                                    + tail(rep, led, alive)))
            if not alive:
                break
    except BreakdownError as err:
        out.append(("breakdown", err, len(out) * stride, led))
    return out


def _cmd_arnoldi_stability(args):
    seed = _seed(args)
    schemes = _schemes(args, SCHEME_IDS)
    op, problem = _operator(args)
    steps = min(args.steps, op.n - 1)
    start = np.random.Generator(np.random.PCG64(seed)).standard_normal(op.n)
    rows = []
    for scheme in schemes:
        for row in _stability_rows(op, start, scheme, steps, args.stride,
                                   lambda rep, led, alive: [str(led.reductions),
                                                            "ok" if alive else "happy-breakdown"]):
            if isinstance(row, tuple):
                _, err, step, led = row
                row = ",".join([scheme, str(step), "nan", "nan", str(led.reductions),
                                f"breakdown-{err.kind}"])
            rows.append(row)
    _write(args, [("schemes", "|".join(schemes)), ("problem", problem), ("steps", steps),
                  ("stride", args.stride), ("seed", seed)],
           "scheme,step,loo,rre,reductions,status", rows)
    return 0


def _cmd_mm_run(args):
    seed = _seed(args)
    schemes = _schemes(args, SCHEME_IDS)
    op, problem = _operator(args)
    steps = min(args.steps, op.n - 1)
    start = np.random.Generator(np.random.PCG64(seed)).standard_normal(op.n)
    tol = args.tol
    rows = []
    for scheme in schemes:
        for row in _stability_rows(op, start, scheme, steps, args.stride,
                                   lambda rep, led, alive: [str(int(rep.loo > tol)),
                                                            str(int(rep.rre > tol)),
                                                            "ok" if alive else "happy-breakdown"]):
            if isinstance(row, tuple):
                _, err, step, _ = row
                row = ",".join([scheme, str(step), "nan", "nan", "1", "1", f"breakdown-{err.kind}"])
            rows.append(row)
    _write(args, [("schemes", "|".join(schemes)), ("problem", problem), ("steps", steps),
                  ("stride", args.stride), ("tol", tol), ("seed", seed)],
           "scheme,step,loo,rre,loo_above_tol,rre_above_tol,status", rows)
    return 0


def _cmd_eig(args):
    seed = _seed(args)
    schemes = _schemes(args, ("cgs2", "dcgs2"))
    restarts = _floats(args.restart_list, cast=int)
    spec = ManteuffelSpec(k=args.manteuffel_k, beta=args.beta)
    csr = manteuffel_build(spec)
    table = manteuffel_eigenvalues(spec)
    rows = []
    for scheme in schemes:
        for restart in restarts:
            cfg = KrylovSchurConfig(max_basis=restart, tol=args.tol, scheme=scheme,
                                    max_restarts=args.max_restarts)
            try:
                res = krylov_schur_run(CsrOperator(csr), cfg, seed=seed, exact=table)
            except BreakdownError as err:
                rows.append(",".join([scheme, str(restart), "-1", "-1", "0",
                                      f"breakdown-{err.kind}"]))
                continue
            rep = match_eigenvalues(res.values.real, table, args.tol)
            status = "over-multiplicity" if res.over_multiplicity else "ok"
            rows.append(",".join([scheme, str(restart), str(rep.n_matched),
                                  str(res.invariant_dim), str(res.restarts), status]))
    _write(args, [("schemes", "|".join(schemes)), ("manteuffel_k", spec.k), ("beta", spec.beta),
                  ("restarts", args.restart_list), ("tol", args.tol),
                  ("max_restarts", args.max_restarts), ("seed", seed)],
           "scheme,restart,n_converged_forward_error,invariant_subspace_dim,restarts_used,status",
           rows)
    return 3 if any(r.endswith("over-multiplicity") for r in rows) else 0


def _cmd_gmres(args):
    seed = _seed(args)
    schemes = _schemes(args, ("cgs2", "dcgs2"))
    if args.mtx:
        op, problem = _operator(args)
    else:
        dims = _floats(args.laplace_dims, cast=int)
        if len(dims) != 3:
            raise _ConfigError("--laplace-dims needs nx,ny,nz")
        op, problem = laplace3d(*dims), f"laplace3d:{dims}"
    b = op.apply(np.ones(op.n)).cpu().numpy()
    b = b / np.linalg.norm(b)
    op.napply = 0
    rows = []
    for scheme in schemes:
        led = SyncLedger()
        res = gmres_solve(op, b, GmresConfig(max_iters=args.steps, restart=args.restart,
                                             scheme=scheme), ledger=led)
        for i in range(len(res.residual_history)):
            rows.append(",".join([scheme, str(i + 1), _fmt(float(res.residual_history[i])),
                                  _fmt(float(res.backward_errors[i])),
                                  str(int(res.reduction_history[i])),
                                  "stagnated" if res.stagnated else "ok"]))
    _write(args, [("schemes", "|".join(schemes)), ("problem", problem), ("iters", args.steps),
                  ("restart", args.restart), ("seed", seed)],
           "scheme,iter,relres,backward_error,reductions,status", rows)
    return 0


def _cmd_sync_count(args):
    seed = _seed(args)
    schemes = _schemes(args, SCHEME_IDS)
    a = np.random.Generator(np.random.PCG64(seed)).standard_normal((args.rows, args.cols))
    rows = []
    failed = False
    for scheme in schemes:
        led = SyncLedger()
        qr_factorize(a, scheme, ledger=led)
        if args.inject_off_by_one:
            led.reductions += 1
        rep = assert_matches(led, predicted_counts(scheme, args.cols))
        failed = failed or not rep.passed
        rows.append(",".join([scheme, str(args.cols), str(args.rows), str(rep.measured),
                              str(rep.predicted), str(rep.slack), str(rep.delta),
                              "pass" if rep.passed else "FAIL"]))
    _write(args, [("schemes", "|".join(schemes)), ("rows", args.rows), ("cols", args.cols),
                  ("seed", seed)],
           "scheme,n,m,measured,predicted,slack,delta,status", rows)
    return 3 if failed else 0


# ---------------------------------------------------------------------------


def build_parser():
    ap = argparse.ArgumentParser(prog="kls-bench",
                                 description="stability and synchronization-cost experiments "
                                             "(B200 backend)")
    ap.add_argument("--version", action="version", version=__version__)
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--scheme", action="append", help="scheme id (repeatable)")
        p.add_argument("--seed", type=int, default=None)
        p.add_argument("--out", default=None)
        p.add_argument("--jobs", type=int, default=1)

    p = sub.add_parser("qr-stability")
    common(p)
    p.add_argument("--kappa-list", default="1e0,1e2,1e4,1e6,1e8,1e10,1e12")
    p.add_argument("--rows", type=int, default=200)
    p.add_argument("--cols", type=int, default=50)
    p.set_defaults(func=_cmd_qr_stability)

    for name, func, steps in (("arnoldi-stability", _cmd_arnoldi_stability, 300),
                              ("mm-run", _cmd_mm_run, 75)):
        p = sub.add_parser(name)
        common(p)
        p.add_argument("--manteuffel-k", type=int, default=50)
        p.add_argument("--beta", type=float, default=0.5)
        p.add_argument("--mtx", default=None, required=(name == "mm-run"))
        p.add_argument("--steps", type=int, default=steps)
        p.add_argument("--stride", type=int, default=5)
        if name == "mm-run":
            p.add_argument("--tol", type=float, default=1e-7)
        p.set_defaults(func=func)

    p = sub.add_parser("eig")
    common(p)
    p.add_argument("--manteuffel-k", type=int, default=10)
    p.add_argument("--beta", type=float, default=0.5)
    p.add_argument("--restart-list", default="25,50,75")
    p.add_argument("--tol", type=float, default=1e-7)
    p.add_argument("--max-restarts", type=int, default=40)
    p.set_defaults(func=_cmd_eig)

    p = sub.add_parser("gmres")
    common(p)
    p.add_argument("--laplace-dims", default="24,24,24")
    p.add_argument("--mtx", default=None)
    p.add_argument("--manteuffel-k", type=int, default=50)
    p.add_argument("--beta", type=float, default=0.5)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--restart", type=int, default=0)
    p.set_defaults(func=_cmd_gmres)

    p = sub.add_parser("sync-count")
    common(p)
    p.add_argument("--rows", type=int, default=5000)
    p.add_argument("--cols", type=int, default=50)
    p.add_argument("--inject-off-by-one", action="store_true", help=argparse.SUPPRESS)
    p.set_defaults(func=_cmd_sync_count)
    return ap


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (_ConfigError, DimensionError, ValueError) as err:
        if isinstance(err, MatrixMarketError) or isinstance(err, (_ConfigError, DimensionError)):
            print(f"error: {err}", file=sys.stderr)
            return 2
        raise
    except BreakdownError as err:
        print(f"error: breakdown halted the run: {err}", file=sys.stderr)
        return 4


if __name__ == "__main__":
    sys.exit(main())
