"""Config 1 per-step time: the round-1 package (scripts/exp/r1pkg, not in
git) against the current one, same box.  python scripts/exp/c1_ab.py r1|new"""
import json, os, sys, time
import numpy as np, torch
HERE = os.path.dirname(os.path.abspath(__file__))
which = sys.argv[1]
sys.path.insert(0, os.path.join(HERE, "r1pkg") if which == "r1" else os.path.dirname(os.path.dirname(HERE)))
import paper_2104_01253_b200 as kls
print(kls.__file__, file=sys.stderr)
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
res = {"pkg": which}
for scheme in ("dcgs2", "cgs2"):
    for _ in range(5):
        kls.arnoldi_expand(op, start, scheme, 50)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(30):
        kls.arnoldi_expand(op, start, scheme, 50)
    torch.cuda.synchronize()
    res[scheme + "_us_per_step"] = round((time.perf_counter() - t0) / 30 / 50 * 1e6, 2)
print(json.dumps(res))
