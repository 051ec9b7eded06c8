"""Config 5's Arnoldi form (band_random_operator m=2.5e7, n=100) timing."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
m = int(sys.argv[1]) if len(sys.argv) > 1 else 25_000_000
op = kls.band_random_operator(m, band=1000, per_row=7, seed=2525)
start = torch.from_numpy(np.random.Generator(np.random.PCG64(1729)).standard_normal(m)).cuda()
kls.arnoldi_expand(op, start, "dcgs2", 100)
ts = []
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    V, H = kls.arnoldi_expand(op, start, "dcgs2", 100)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print(json.dumps({"config": "5a", "m": m, "fused": os.environ.get("KLS_FUSED", "1"), "s": min(ts),
                  "it_s": 100 / min(ts), "H_sum": float(np.abs(H).sum())}))
