"""Where config 1's expansion time goes (m = 1e4, n = 50): cProfile of
repeated arnoldi_expand calls, top entries by cumulative time."""
import cProfile, io, os, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for _ in range(5):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
print("us per expansion", (time.perf_counter() - t0) / 50 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(50):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25); print(s.getvalue()[:6000])
