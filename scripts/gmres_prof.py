"""cProfile of restarted GMRES at config-2 size (m = 1e6, restart 50)."""
import cProfile, io, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as kls
op = kls.manteuffel_operator(kls.ManteuffelSpec(k=1000, beta=0.5))
one = op.apply(np.ones(op.n)).cpu().numpy()
b = one / np.linalg.norm(one)
for be in (False, True):
    cfg = kls.GmresConfig(max_iters=600, restart=50, rtol=1e-12, scheme="dcgs2", backward_errors=be)
    kls.gmres_solve(op, b, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = kls.gmres_solve(op, b, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print("backward_errors", be, "iterations", res.iterations, "us/it", dt / res.iterations * 1e6)
pr = cProfile.Profile(); pr.enable()
kls.gmres_solve(op, b, kls.GmresConfig(max_iters=600, restart=50, rtol=1e-12, scheme="dcgs2", backward_errors=False))
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(22); print(s.getvalue()[:5000])
