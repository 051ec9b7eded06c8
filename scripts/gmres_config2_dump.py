"""Run BASELINE config 2 (GMRES(50), DCGS2, m = 1e6, rtol 1e-6) on the GPU and
save the residual history to gpurun_out/gc2_gpu.npz (for comparing against
tests/golden/gmres_config2.npz and the reference's own self-noise)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as K

op = K.CsrOperator(K.manteuffel_build(K.ManteuffelSpec(k=1000, beta=0.5)))
one = op.apply(np.ones(op.n)).cpu().numpy()
b = one / np.linalg.norm(one)
res = K.gmres_solve(op, b, K.GmresConfig(max_iters=10000, restart=50, rtol=1e-6, scheme="dcgs2"))
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/gc2_gpu.npz", iterations=res.iterations,
                    residual_history=res.residual_history)
print(res.iterations)
