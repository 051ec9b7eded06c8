"""Config 1 (m = 1e4, n = 50, DCGS2): per-expansion time untraced, and the
traced per-kernel device time per step; then the Gram kernel alone
(kls_gram_dcgs2_step at j = 25, back to back)."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
from paper_2104_01253_b200 import _lib, runtime, trace
op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
start = np.random.Generator(np.random.PCG64(1729)).standard_normal(op.n)
for _ in range(5):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    kls.arnoldi_expand(op, start, "dcgs2", 50)
torch.cuda.synchronize()
per = (time.perf_counter() - t0) / 20
rec = trace.start(events=True)
kls.arnoldi_expand(op, start, "dcgs2", 50)
trace.stop()
spans = {k: round(rec.seconds(k) / 50 * 1e6, 2) for k in ("gram", "update", "project", "mtm", "apply", "scale")
         if rec.seconds(k) > 0}
m, ld, j = op.m_local, runtime.pad_rows(op.m_local), 25
Q = torch.randn((51, ld), dtype=torch.float64, device="cuda")
w = torch.randn(ld, dtype=torch.float64, device="cuda")
aw = torch.randn(ld, dtype=torch.float64, device="cuda")
g = torch.empty(128, dtype=torch.float64, device="cuda")
c = torch.empty(128, dtype=torch.float64, device="cuda")
ws, wsb = runtime.workspace(64)
st = runtime.stream_handle()
def gram():
    _lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(), g.data_ptr(),
              c.data_ptr(), None, 0, op.segs.ptr, ws, wsb, st)
for _ in range(10): gram()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(500): gram()
e1.record(); torch.cuda.synchronize()
print(json.dumps({"ms_per_expansion": round(per * 1e3, 3), "us_per_step": round(per / 50 * 1e6, 2),
                  "traced_us_per_step": spans, "gram_step_j25_us": round(e0.elapsed_time(e1) * 1e3 / 500, 2)}))
