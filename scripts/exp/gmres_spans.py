"""Per-kernel device time of restarted GMRES at config 2 (m = 1e6, restart 50)
with and without per-column backward errors: the event tracer's spans plus
an untraced wall/event time, 600 iterations.  The ell_resid_norms launches
(fused backward-error column) are timed by a separate probe: N launches back
to back at m = 1e6."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
from paper_2104_01253_b200 import _lib, runtime, trace
op = kls.manteuffel_operator(kls.ManteuffelSpec(k=1000, beta=0.5))
one = op.apply(torch.ones(op.m_local, dtype=torch.float64, device="cuda"))
b = one / kls.kernels.norm2(one, comm=op.comm, segs=op.segs)
for be in (False, True):
    cfg = kls.GmresConfig(max_iters=600, restart=50, rtol=1e-12, scheme="dcgs2", backward_errors=be)
    kls.gmres_solve(op, b, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = kls.gmres_solve(op, b, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rec = trace.start(events=True)
    kls.gmres_solve(op, b, cfg)
    trace.stop()
    spans = {k: round(rec.seconds(k) / res.iterations * 1e6, 2) for k in
             ("gram", "update", "project", "project_gram", "mtm", "apply", "resid_norms", "scale")
             if rec.seconds(k) > 0}
    print(json.dumps({"backward_errors": be, "iterations": res.iterations,
                      "us_per_it_untraced": round(dt / res.iterations * 1e6, 2),
                      "us_per_it_traced_kernels": spans}), flush=True)
ecol, evals, elen, width, ld = op._ell
x = torch.randn(op.m_local, dtype=torch.float64, device="cuda")
out = torch.empty(3, dtype=torch.float64, device="cuda")
ws, wsb = runtime.workspace(64)
st = runtime.stream_handle()
for _ in range(3):
    _lib.call("kls_ell_resid_norms", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width,
              op.m_local, ld, x.data_ptr(), b.data_ptr(), out.data_ptr(), op.segs.ptr, ws, wsb, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    _lib.call("kls_ell_resid_norms", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width,
              op.m_local, ld, x.data_ptr(), b.data_ptr(), out.data_ptr(), op.segs.ptr, ws, wsb, st)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"ell_resid_norms_us": round(e0.elapsed_time(e1) * 1e3 / 200, 2),
                  "bytes_GBs": round((16 * op.m_local + 13 * width * op.m_local) / (e0.elapsed_time(e1) / 200 * 1e-3) / 1e9, 1)}))
