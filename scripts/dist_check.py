"""Multi-GPU parity check (torchrun, one process per GPU, NCCL):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/dist_check.py

Row-sharded DCGS2 / CGS2 Arnoldi on the matrix-free stencil and on a CSR
operator, plus restarted GMRES, compared on rank 0 with the CPU oracle run
single-process on the same global input, and config 3's expansion shape
and config 2 at full size against the reference's own runs
(tests/golden/arnoldi_config3_shape.npz, gmres_config2.npz).
Prints one JSON line; exit 1 on a parity failure.
"""

import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2104_01253_b200 import runtime

    comm = runtime.init_distributed()  # ranks may share GPUs (gloo + CUDA-IPC peers)
    rank, world = comm.rank, comm.world
    import oracle
    import paper_2104_01253_b200 as kls

    res = {"world": world}
    ok = True

    def gather_h(H):
        return H  # host math is replicated: every rank holds the same H

    # stencil, both schemes
    dims = (40, 30, 20)
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(int(np.prod(dims)))
    for scheme in ("dcgs2", "cgs2"):
        op = kls.laplace3d(*dims)
        led = kls.SyncLedger()
        V, H = kls.arnoldi_expand(op, start, scheme, steps=30, ledger=led)
        loo = kls.loss_of_orthogonality(V, segs=op.segs)
        if rank == 0:
            _, Hr, cnt = getattr(oracle, f"{scheme}_arnoldi")(
                lambda x: oracle.stencil7_matvec(x, dims), start, 30)
            err = float(np.max(np.abs(H - Hr)) / np.max(np.abs(Hr)))
            res[f"stencil_{scheme}_relerr"] = err
            res[f"stencil_{scheme}_loo"] = loo
            res[f"stencil_{scheme}_reductions"] = [led.reductions, cnt.reductions]
            ok &= err <= 1e-10 and led.reductions == cnt.reductions and loo <= 1e-12
    # config 3's expansion shape against the reference's own run (golden)
    g = np.load(os.path.join(ROOT, "tests", "golden", "arnoldi_config3_shape.npz"))
    start3 = np.random.Generator(np.random.PCG64(1729)).standard_normal(62 * 64 * 64)
    for scheme in ("dcgs2", "cgs2"):
        op = kls.laplace3d(62, 64, 64)
        led = kls.SyncLedger()
        V, H = kls.arnoldi_expand(op, start3, scheme, steps=100, ledger=led)
        loo = kls.loss_of_orthogonality(V, segs=op.segs)
        ref = g[f"{scheme}_H"]
        err = float(np.max(np.abs(H - ref)) / np.max(np.abs(ref)))
        if rank == 0:
            res[f"config3_shape_{scheme}_relerr"] = err
            res[f"config3_shape_{scheme}_loo"] = loo
        ok &= (err <= 1e-10 and led.reductions == int(g[f"{scheme}_reductions"]) and
               loo <= 10 * max(float(g[f"{scheme}_loo"]), 1e-15))
    # CSR (Manteuffel k=60)
    k = 60
    csr = kls.manteuffel_build(kls.ManteuffelSpec(k=k))
    start = np.random.Generator(np.random.PCG64(7)).standard_normal(k * k)
    op = kls.CsrOperator(csr)
    V, H = kls.arnoldi_expand(op, start, "dcgs2", steps=30)
    if rank == 0:
        ptr, idx, dat = oracle.manteuffel_csr(k, 0.5)
        _, Hr, _ = oracle.dcgs2_arnoldi(lambda x: oracle.csr_matvec(ptr, idx, dat, x), start, 30)
        err = float(np.max(np.abs(H - Hr)) / np.max(np.abs(Hr)))
        res["csr_dcgs2_relerr"] = err
        ok &= err <= 1e-10
    # device-built CSR operators (row-sharded assembly in HBM)
    dims2 = (12, 10, 9)
    start2 = np.random.Generator(np.random.PCG64(11)).standard_normal(int(np.prod(dims2)))
    _, Hd = kls.arnoldi_expand(kls.laplace3d_csr_operator(*dims2), start2, "dcgs2", steps=25)
    _, Hs = kls.arnoldi_expand(kls.laplace3d(*dims2), start2, "dcgs2", steps=25)
    kk = 40
    startm = np.random.Generator(np.random.PCG64(12)).standard_normal(kk * kk)
    _, Hm = kls.arnoldi_expand(kls.manteuffel_operator(kls.ManteuffelSpec(k=kk)), startm, "dcgs2", 25)
    if rank == 0:
        e1 = float(np.max(np.abs(Hd - Hs)) / np.max(np.abs(Hs)))
        ptr, idx, dat = oracle.manteuffel_csr(kk, 0.5)
        _, Hr, _ = oracle.dcgs2_arnoldi(lambda x: oracle.csr_matvec(ptr, idx, dat, x), startm, 25)
        e2 = float(np.max(np.abs(Hm - Hr)) / np.max(np.abs(Hr)))
        res["device_csr_lap_vs_stencil"] = e1
        res["device_csr_mant_vs_oracle"] = e2
        ok &= e1 <= 1e-12 and e2 <= 1e-10
    # GMRES
    k = 30
    csr = kls.manteuffel_build(kls.ManteuffelSpec(k=k))
    op = kls.CsrOperator(csr)
    ptr, idx, dat = oracle.manteuffel_csr(k, 0.5)
    one = oracle.csr_matvec(ptr, idx, dat, np.ones(k * k))
    b = one / np.linalg.norm(one)
    g = kls.gmres_solve(op, b, kls.GmresConfig(max_iters=300, restart=20, rtol=1e-8,
                                               scheme="dcgs2"))
    if rank == 0:
        r = oracle.gmres(lambda x: oracle.csr_matvec(ptr, idx, dat, x), b,
                         float(np.linalg.norm(dat)), 300, 20, 1e-8, "dcgs2")
        res["gmres_iterations"] = [g.iterations, r["iterations"]]
        nn = min(len(g.residual_history), len(r["residual_history"]))
        dh = np.abs(g.residual_history[:nn] - r["residual_history"][:nn])
        res["gmres_first_bad"] = int(np.argmax(dh > 1e-8)) if np.any(dh > 1e-8) else -1
        res["gmres_hist"] = [g.residual_history[:45:4].tolist(), r["residual_history"][:45:4].tolist()]
        res["gmres_be"] = [g.backward_errors[:45:4].tolist(), r["backward_errors"][:45:4].tolist()]
        dev = float(np.max(dh)) if g.iterations == r["iterations"] else float("inf")
        res["gmres_hist_maxdiff"] = dev
        ok &= g.iterations == r["iterations"] and dev <= 1e-8
    # config 2 at full size (m = 1e6, GMRES(50), rtol 1e-6) row-sharded,
    # against the reference's own run (tests/golden/gmres_config2.npz)
    g2 = np.load(os.path.join(ROOT, "tests", "golden", "gmres_config2.npz"))
    ptr2, idx2, dat2 = oracle.manteuffel_csr(1000, 0.5)
    one2 = oracle.csr_matvec(ptr2, idx2, dat2, np.ones(1000 * 1000))
    b2 = one2 / np.linalg.norm(one2)
    op2 = kls.manteuffel_operator(kls.ManteuffelSpec(k=1000, beta=0.5))
    led2 = kls.SyncLedger()
    gm = kls.gmres_solve(op2, b2, kls.GmresConfig(max_iters=10000, restart=50, rtol=1e-6,
                                                  scheme="dcgs2"), ledger=led2)
    ref2 = g2["residual_history"]
    spread2 = np.abs(g2["residual_history_threads8"] - ref2)
    same_len = gm.residual_history.shape == ref2.shape
    dev2 = float(np.max(np.abs(gm.residual_history - ref2))) if same_len else float("inf")
    if rank == 0:
        res["config2_iterations"] = [gm.iterations, int(g2["iterations"])]
        res["config2_hist_maxdiff"] = dev2
    ok &= (gm.iterations == int(g2["iterations"]) and led2.reductions == int(g2["reductions"])
           and dev2 <= 3.0 * float(spread2.max()))
    # DCGS2 / CGS2 QR of a row-sharded tall-skinny matrix (config 5's kernel)
    A = np.random.Generator(np.random.PCG64(21)).standard_normal((50_021, 24))
    for scheme in ("dcgs2", "cgs2"):
        led = kls.SyncLedger()
        Qd, R = kls.qr_factorize(A, scheme, ledger=led)
        loo = kls.loss_of_orthogonality(Qd, segs=comm.segs(A.shape[0]))
        if rank == 0:
            _, Rr, cnt = getattr(oracle, f"{scheme}_qr")(A)
            err = float(np.max(np.abs(R - Rr)) / np.max(np.abs(Rr)))
            res[f"qr_{scheme}_relerr"] = err
            ok &= err <= 1e-10 and loo <= 1e-13 and led.reductions == cnt.reductions
    # Krylov-Schur on the row-sharded operator: every locked value must be an
    # exact eigenvalue (manteuffel_eigenvalues) with the right multiplicity,
    # the lock history identical on all ranks, Ritz vectors sharded
    spec = kls.ManteuffelSpec(k=8)
    op = kls.CsrOperator(kls.manteuffel_build(spec))
    table = kls.manteuffel_eigenvalues(spec)
    ks = kls.krylov_schur_run(op, kls.KrylovSchurConfig(max_basis=30, tol=1e-7, scheme="dcgs2",
                                                        max_restarts=8), seed=11, exact=table)
    hist = [None] * world
    dist.all_gather_object(hist, ks.lock_history)
    rep = kls.match_eigenvalues(ks.values.real, table, 1e-7)
    res["ks_locked"] = ks.invariant_dim
    res["ks_matched"] = rep.n_matched
    ok &= (all(h == hist[0] for h in hist) and ks.invariant_dim > 0
           and rep.n_matched == len(ks.values) and not ks.over_multiplicity
           and ks.vectors.shape[0] == op.m_local)
    res["ok"] = bool(ok)
    flag = -comm.allreduce_max_float(-(1.0 if ok or rank != 0 else 0.0))
    if rank == 0:
        print(json.dumps(res), flush=True)
    runtime.shutdown_distributed()
    return 0 if flag == 1.0 else 1


if __name__ == "__main__":
    sys.exit(main())
