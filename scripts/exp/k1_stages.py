"""K1 (kls_gram_dcgs2, the TMA-staged Gram pass) device time at medium and
headline m.  Prints one JSON line.  Used with a temporary KLS_K1_STAGES
ring-depth knob (3-6 stages: within 2 %; the knob was removed and
the ring stays at 4 stages)."""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2104_01253_b200 import _lib as lib, runtime as rt

out = {"stages": os.environ.get("KLS_K1_STAGES", "4")}
for m, js in ((1_000_000, (10, 25, 50)), (10_000_000, (30, 60)), (130_023_424, (25, 50, 100))):
    jmax = max(js)
    ld = rt.pad_rows(m)
    Q = torch.empty((jmax, ld), dtype=torch.float64, device="cuda").normal_()
    w = torch.randn(m, dtype=torch.float64, device="cuda")
    aw = torch.randn(m, dtype=torch.float64, device="cuda")
    g = torch.empty(2 * jmax + 3, dtype=torch.float64, device="cuda")
    ws, wsb = rt.workspace(jmax + 2)
    st = rt.stream_handle()
    for j in js:
        f = lambda: lib.call("kls_gram_dcgs2", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
                             g.data_ptr(), None, ws, wsb, st)
        for _ in range(3):
            f()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); f(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        t = float(np.median(ts))
        out[f"m{m}_j{j}"] = {"us": round(t, 1), "GBs": round(8 * m * (j + 2) / t / 1e3)}
    del Q, w, aw
    torch.cuda.empty_cache()
print(json.dumps(out))
