"""cProfile of Krylov-Schur at config-4 size: where a restart spends its time.

    python scripts/ks_probe.py [k=3163] [restarts=400]
"""
import cProfile, io, json, os, pstats, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as kls
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3163
R = int(sys.argv[2]) if len(sys.argv) > 2 else 400
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=k, beta=0.5)))
cfg = kls.KrylovSchurConfig(max_basis=60, tol=1e-7, scheme="dcgs2", max_restarts=R)
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); res = kls.krylov_schur_run(op, cfg, seed=1729); torch.cuda.synchronize(); t = time.perf_counter() - t0
pr.disable()
print(json.dumps({"k": k, "m": op.n, "restarts": res.restarts, "nlock": res.invariant_dim, "s": t,
                  "hist_tail": res.lock_history[-10:], "first_locked": [str(v) for v in res.values[:10]]}))
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumtime").print_stats(18); print(s.getvalue()[:3500])
