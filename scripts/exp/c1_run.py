import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2104_01253_b200 as kls
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
s = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for _ in range(3):
    kls.arnoldi_expand(op, s, "dcgs2", 50)
