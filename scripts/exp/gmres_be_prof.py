"""Host-side profile of GMRES(50) with per-column backward errors at m = 1e6
(config 2): is the loop host- or GPU-bound?"""
import cProfile, io, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
op = kls.manteuffel_operator(kls.ManteuffelSpec(k=1000, beta=0.5))
one = op.apply(np.ones(op.n)).cpu().numpy()
b = one / np.linalg.norm(one)
cfg = kls.GmresConfig(max_iters=600, restart=50, rtol=1e-12, scheme="dcgs2", backward_errors=True)
kls.gmres_solve(op, b, cfg)
torch.cuda.synchronize()
t0 = time.perf_counter(); res = kls.gmres_solve(op, b, cfg); torch.cuda.synchronize()
print("us/it", (time.perf_counter() - t0) / res.iterations * 1e6)
pr = cProfile.Profile(); pr.enable()
kls.gmres_solve(op, b, cfg); torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
