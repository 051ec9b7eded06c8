"""GPU time of one lookahead step's launch chain (K2 update -> operator ->
K1 Gram + scalar step, one kls_dcgs2_queue_step call) at config 1's size,
queued back to back without host waits: compare with the per-step time of a
real expansion (which adds the host's wait + host step) to see whether the
small-m step is GPU- or host-bound.

    python scripts/chain_step_probe.py
"""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_01253_b200 as kls

op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for j in (5, 25, 45):
    exp = kls.arnoldi(op, start, "dcgs2", 51)
    for _ in range(j):
        exp.step()
    e = exp.eng
    plan = e.step_plan()
    w, aw, w2, aw2 = exp._w, exp._aw, exp._w2, exp._aw2
    for _ in range(20):
        e.queue_step(plan, j, w.local, w2, aw, aw2, 0, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 300
    t0 = time.perf_counter()
    e0.record(torch.cuda.current_stream())
    for _ in range(n):
        e.queue_step(plan, j, w.local, w2, aw, aw2, 0, True)
    e1.record(torch.cuda.current_stream())
    host = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print({"j": j, "gpu_us_per_step": round(e0.elapsed_time(e1) * 1e3 / n, 2),
           "host_queue_us_per_step": round(host, 2)})
# a real expansion: steps/s over 50 steps
for _ in range(3):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
print({"expansion_us_per_step": round((time.perf_counter() - t0) / 20 / 50 * 1e6, 2)})
