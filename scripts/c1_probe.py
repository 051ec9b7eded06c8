"""Config-1-sized DCGS2 expansions (m = 1e4, 50 steps) for an ncu launch list:

    ncu --metrics gpu__time_duration.sum --csv python scripts/c1_probe.py
"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2104_01253_b200 as kls
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for _ in range(3): kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
