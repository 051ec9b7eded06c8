"""Run BASELINE.json configs 1, 2, 4 and 5 on one GPU and (bounded) on the
host CPU reference; print one JSON line per measurement.

    python scripts/configs.py [--only 1,2,4,5] [--cpu]

Config 3 is bench.py's headline.  CPU timings use the unmodified reference
from baseline/_ref (kind "reference") on bounded samples stated per line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2104_01253_b200 as kls  # noqa: E402


def ref():
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    import kls as R

    return R


def gtime(fn, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, out


def emit(d):
    print(json.dumps(d), flush=True)


def config1(cpu):
    op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
    for scheme in ("dcgs2", "cgs2"):
        kls.arnoldi_expand(op, start, scheme, 50)
        t, _ = gtime(lambda: kls.arnoldi_expand(op, start, scheme, 50), reps=20)
        d = {"config": 1, "scheme": scheme, "m": op.n, "n": 50, "gpu_s": t, "gpu_it_s": 50 / t}
        if cpu:
            R = ref()
            rop = R.CsrOperator(R.manteuffel_build(R.ManteuffelSpec(k=100, beta=0.0)))
            t0 = time.perf_counter()
            for _ in range(3):
                R.arnoldi_expand(rop, start, scheme, 50)
            tc = (time.perf_counter() - t0) / 3
            d.update(cpu_s=tc, cpu_it_s=50 / tc, speedup=tc / t)
        emit(d)


def config2(cpu, max_iters):
    spec = kls.ManteuffelSpec(k=1000, beta=0.5)
    csr = kls.manteuffel_build(spec)
    op = kls.CsrOperator(csr)
    one = op.apply(np.ones(op.n)).cpu().numpy()
    b = one / np.linalg.norm(one)
    for be in (True, False):
        cfg = kls.GmresConfig(max_iters=max_iters, restart=50, rtol=1e-6, scheme="dcgs2",
                              backward_errors=be)
        kls.gmres_solve(op, b, cfg)  # warm-up (engine buffers, stream, caches)
        led = kls.SyncLedger()
        t, res = gtime(lambda: kls.gmres_solve(op, b, cfg, ledger=led))
        d = {"config": 2, "m": op.n, "restart": 50, "rtol": 1e-6, "backward_errors": be,
             "iterations": res.iterations, "converged": res.converged,
             "final_relres": float(res.residual_history[-1]), "gpu_s": t,
             "gpu_it_s": res.iterations / t, "reductions": led.reductions}
        emit(d)
    if cpu:
        R = ref()
        rop = R.CsrOperator(R.manteuffel_build(R.ManteuffelSpec(k=1000, beta=0.5)))
        t0 = time.perf_counter()
        rr = R.gmres_solve(rop, b, R.GmresConfig(max_iters=100, restart=50, rtol=1e-6,
                                                 scheme="dcgs2"))
        tc = time.perf_counter() - t0
        emit({"config": 2, "cpu_sample": "reference gmres_solve, first 100 iterations",
              "cpu_s": tc, "cpu_it_s": rr.iterations / tc,
              "relres_100": float(rr.residual_history[-1])})


def config4(cpu, restarts):
    spec = kls.ManteuffelSpec(k=3163, beta=0.5)
    t0 = time.perf_counter()
    csr = kls.manteuffel_build(spec)
    op = kls.CsrOperator(csr)
    build = time.perf_counter() - t0
    cfg = kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=restarts)
    t, res = gtime(lambda: kls.krylov_schur_run(op, cfg, seed=1729))
    emit({"config": 4, "m": op.n, "max_basis": 60, "restarts": res.restarts,
          "invariant_dim": res.invariant_dim, "lock_history": res.lock_history,
          "first_locked": [str(v) for v in res.values[:10]], "gpu_s": t,
          "gpu_s_per_restart": t / res.restarts, "host_build_s": build})


def config5(n_list, m):
    for n in n_list:
        g = torch.Generator(device="cuda")
        g.manual_seed(1729)
        A = torch.randn((n, m), generator=g, dtype=torch.float64, device="cuda")
        A *= (torch.rand((n, m), generator=g, device="cuda") < 1e-3)
        cols = [A[j] for j in range(n)]

        def qr():
            st = kls.make_state("dcgs2", m, n)
            for c in cols:
                st.push(c)
            return st.finalize()

        qr()
        t, (Q, R) = gtime(qr)
        loo = kls.loss_of_orthogonality(Q)
        bytes_ = sum(8 * m * (2 * j + 6) for j in range(n))
        emit({"config": 5, "m": m, "n": n, "gpu_s": t, "cols_per_s": n / t,
              "hbm_GBs_algorithmic": bytes_ / t / 1e9, "loo": loo})
        del A, cols, Q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="1,2,4,5")
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--gmres-iters", type=int, default=10000)
    ap.add_argument("--ks-restarts", type=int, default=30)
    ap.add_argument("--qr-m", type=int, default=25_000_000)
    ap.add_argument("--qr-n", default="25,50,100,200")
    a = ap.parse_args()
    only = {int(v) for v in a.only.split(",")}
    if 1 in only:
        config1(a.cpu)
    if 2 in only:
        config2(a.cpu, a.gmres_iters)
    if 4 in only:
        config4(a.cpu, a.ks_restarts)
    if 5 in only:
        config5([int(v) for v in a.qr_n.split(",")], a.qr_m)


if __name__ == "__main__":
    main()
