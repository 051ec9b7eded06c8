"""Per-launch fixed cost of K1 (Gram + fused scalar step) and K2 (update)
at medium m: time each kernel alone, back to back (CUDA events), and report
the excess over the algorithmic bytes at a reference bandwidth.

    SIZES=1e6,1e7 python scripts/fixed_cost_probe.py
"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_01253_b200 import _lib, runtime

BW = 7.3e12
for m in [int(float(v)) for v in os.environ.get("SIZES", "1e6,1e7").split(",")]:
    for j in (1, 8, 25, 50):
        ld = runtime.pad_rows(m)
        Q = torch.randn((j + 1, ld), dtype=torch.float64, device="cuda") / np.sqrt(m)
        w = torch.randn(m, dtype=torch.float64, device="cuda")
        aw = torch.randn(m, dtype=torch.float64, device="cuda")
        w2 = torch.empty_like(w)
        g = torch.empty(2 * j + 3, dtype=torch.float64, device="cuda")
        c = torch.empty(2 * j + 2, dtype=torch.float64, device="cuda")
        ws, wsb = runtime.workspace(j + 2)
        st = runtime.stream_handle()

        def k1():
            _lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
                      g.data_ptr(), c.data_ptr(), None, 0, None, ws, wsb, st)

        def k1plain():
            _lib.call("kls_gram_dcgs2", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
                      g.data_ptr(), None, ws, wsb, st)

        def k2():
            _lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(), w2.data_ptr(),
                      aw.data_ptr(), c.data_ptr(), 1, None, st)

        k1()
        torch.cuda.synchronize()
        c.copy_(torch.rand_like(c) * 0.1 + 1.0)
        out = {"m": m, "j": j}
        for name, fn, nbytes in (("k1", k1, 8 * m * (j + 2)), ("k1_noscalar", k1plain, 8 * m * (j + 2)),
                                 ("k2", k2, 8 * m * (j + 4))):
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 50
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            out[name + "_us"] = round(us, 2)
            out[name + "_excess_us"] = round(us - nbytes / BW * 1e6, 2)
            out[name + "_TBs"] = round(nbytes / us / 1e6, 2)
        print(json.dumps(out), flush=True)
