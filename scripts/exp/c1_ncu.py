"""Config 1 expansion under ncu's launch list: python scripts/exp/c1_ncu.py r1|new"""
import os, sys
import numpy as np, torch
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "r1pkg") if sys.argv[1] == "r1" else os.path.dirname(os.path.dirname(HERE)))
import paper_2104_01253_b200 as kls
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for _ in range(2):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
