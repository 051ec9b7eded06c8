"""A short config-2-sized GMRES run (m = 1e6, restart 50, 200 iterations)
for an ncu launch list of the per-iteration kernels."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as kls
op = kls.manteuffel_operator(kls.ManteuffelSpec(k=1000, beta=0.5))
one = op.apply(np.ones(op.n)).cpu().numpy()
b = one / np.linalg.norm(one)
be = os.environ.get("BE", "0") == "1"
kls.gmres_solve(op, b, kls.GmresConfig(max_iters=200, restart=50, rtol=1e-12, scheme="dcgs2",
                                      backward_errors=be))
torch.cuda.synchronize()
