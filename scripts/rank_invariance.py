"""Rank-count independence of the row-sharded path on the GPU.

Every reduction follows a fixed 24-segment tree, so the same global problem
gives BITWISE the same scalars -- Hessenberg H, QR's R, GMRES iterations and
residual histories, Krylov-Schur lock histories and Ritz values, basis rows
-- on any number of ranks.  Run the cases at each N, then compare:

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/rank_invariance.py \\
        --out gpurun_out/rankinv_N.npz
    python scripts/rank_invariance.py --compare gpurun_out/rankinv_*.npz

The compare step prints one JSON line (per case: equal to the N = 1 run or
the max abs difference) and exits 1 on any difference.  Ranks may share a
GPU (N > device count: device = LOCAL_RANK % count, gloo bootstrap, CUDA-IPC
peer buffers -- runtime.PeerLink).
"""

import argparse
import glob
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _rows(V, op, every):
    """Global rows lo + i of the local basis V with (lo + i) % every == 0,
    gathered on every rank: (row index, row) sorted by row."""
    import torch.distributed as dist

    lo = op.row_lo
    first = (-lo) % every
    idx = np.arange(first, V.shape[0], every)
    mine = (lo + idx, V[idx.tolist()].cpu().numpy() if idx.size else np.zeros((0, V.shape[1])))
    got = [None] * dist.get_world_size() if dist.is_initialized() else [mine]
    if dist.is_initialized():
        dist.all_gather_object(got, mine)
    rows = np.concatenate([g[0] for g in got])
    vals = np.concatenate([g[1] for g in got])
    order = np.argsort(rows)
    return vals[order]


def run(out_path):
    import torch

    from paper_2104_01253_b200 import runtime

    comm = runtime.init_distributed()
    import paper_2104_01253_b200 as kls

    res = {"world": comm.world}

    # config 3's expansion shape (3-D Poisson, x-plane partition), both schemes
    start3 = np.random.Generator(np.random.PCG64(1729)).standard_normal(62 * 64 * 64)
    for scheme in ("dcgs2", "cgs2"):
        op = kls.laplace3d(62, 64, 64)
        led = kls.SyncLedger()
        V, H = kls.arnoldi_expand(op, start3, scheme, steps=100, ledger=led)
        res[f"stencil_{scheme}_H"] = H
        res[f"stencil_{scheme}_Vrows"] = _rows(V, op, 4999)
        res[f"stencil_{scheme}_reductions"] = led.reductions
    # host CSR (Manteuffel, config 4's operator family) and a device-built one
    start = np.random.Generator(np.random.PCG64(7)).standard_normal(100 * 100)
    op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.5)))
    V, H = kls.arnoldi_expand(op, start, "dcgs2", steps=60)
    res["csr_H"], res["csr_Vrows"] = H, _rows(V, op, 997)
    startd = np.random.Generator(np.random.PCG64(8)).standard_normal(300 * 300)
    opd = kls.manteuffel_operator(kls.ManteuffelSpec(k=300, beta=0.5))
    _, H = kls.arnoldi_expand(opd, startd, "dcgs2", steps=50)
    res["device_csr_H"] = H
    # restarted GMRES (per-column backward errors on)
    one = op.apply(torch.ones(op.m_local, dtype=torch.float64, device="cuda"))
    nrm = kls.kernels.norm2(one, comm=op.comm, segs=op.segs)
    b = one / nrm
    g = kls.gmres_solve(op, b, kls.GmresConfig(max_iters=3000, restart=50, rtol=1e-8,
                                               scheme="dcgs2"))
    res["gmres_iterations"] = g.iterations
    res["gmres_residual_history"] = g.residual_history
    res["gmres_backward_errors"] = g.backward_errors
    # Krylov-Schur at config 4's settings (m = 1e4, 30 restarts)
    ks = kls.krylov_schur_run(op, kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2",
                                                        max_restarts=30), seed=1729)
    res["ks_lock_history"] = np.array(ks.lock_history)
    res["ks_values"] = np.asarray(ks.values)
    # DCGS2 / CGS2 QR of a tall-skinny block (config 5's kernel)
    A = np.random.Generator(np.random.PCG64(21)).standard_normal((50_021, 24))
    for scheme in ("dcgs2", "cgs2"):
        Qd, R = kls.qr_factorize(A, scheme)
        res[f"qr_{scheme}_R"] = R
    if comm.rank == 0:
        os.makedirs(os.path.dirname(os.path.abspath(out_path)), exist_ok=True)
        np.savez(out_path, **res)
        print(json.dumps({"world": comm.world, "saved": out_path,
                          "gmres_iterations": int(g.iterations),
                          "ks_lock_history_tail": [int(x) for x in ks.lock_history[-5:]]}),
              flush=True)
    runtime.shutdown_distributed()


def compare(paths):
    runs = {}
    for p in paths:
        d = np.load(p)
        runs[int(d["world"])] = d
    base = runs[1]
    out = {"worlds": sorted(runs), "cases": {}}
    ok = True
    for key in base.files:
        if key == "world":
            continue
        row = {}
        for w in sorted(runs):
            if w == 1:
                continue
            a, b = base[key], runs[w][key]
            same = a.shape == b.shape and np.array_equal(a, b)
            if same:
                row[str(w)] = "equal"
            else:
                ok = False
                row[str(w)] = (float(np.max(np.abs(a - b))) if a.shape == b.shape
                               else f"shape {a.shape} vs {b.shape}")
        out["cases"][key] = row
    out["ok"] = ok
    print(json.dumps(out))
    return 0 if ok else 1


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out")
    ap.add_argument("--compare", nargs="*")
    a = ap.parse_args()
    if a.compare is not None:
        paths = [p for g in a.compare for p in glob.glob(g)]
        sys.exit(compare(paths))
    run(a.out)
