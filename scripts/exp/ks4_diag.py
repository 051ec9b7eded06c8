"""Row-sharded Krylov-Schur at config 4's settings (m = 1e4, max_basis 60,
tol 1e-7, 30 restarts) against the reference's run: prints the lock history
beside the golden one.  torchrun --nproc-per-node N scripts/exp/ks4_diag.py"""
import os, sys, json
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, "/root/repo")
from paper_2104_01253_b200 import runtime
runtime.init_distributed()
import paper_2104_01253_b200 as kls
g4 = np.load("/root/repo/tests/golden/ks_config4_shape.npz")
op4 = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.5)))
ks4 = kls.krylov_schur_run(op4, kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=30), seed=1729)
if dist.get_rank() == 0:
    ref, alt = g4["values"], g4["alt_values"]
    out = {"world": dist.get_world_size(), "hist": [int(x) for x in ks4.lock_history], "ref_hist": [int(x) for x in g4["lock_history"]]}
    if ks4.values.shape == ref.shape:
        rel = np.abs(ks4.values - ref) / np.abs(ref); drift = np.abs(alt - ref) / np.abs(ref)
        out["max_rel"] = float(rel.max()); out["ratio_max"] = float(np.max(rel / np.maximum(1e-9, drift)))
    print(json.dumps(out))
runtime.shutdown_distributed()
