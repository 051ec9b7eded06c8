"""cProfile of the host side of small-m expansions (config 1 size)."""
import cProfile, io, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as kls
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for _ in range(3): kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
print("per step us", (time.perf_counter()-t0)/20/50*1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
