"""Warm-cache latency of the Gram (K1, fused scalar step) and update (K2)
kernels at small m: CUDA events around 200 back-to-back launches.

    python scripts/small_probe.py            # KLS_GRAM=big / KLS_UPDATE=ldg to compare
"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_01253_b200 import _lib, runtime

def bench(fn, reps=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps

for m in [int(float(v)) for v in os.environ.get("SIZES", "1e4,1e5,1e6").split(",")]:
    for j in (10, 50, 100):
        ld = runtime.pad_rows(m)
        Q = torch.randn((j + 1, ld), dtype=torch.float64, device="cuda") / np.sqrt(m)
        w = torch.randn(m, dtype=torch.float64, device="cuda")
        aw = torch.randn(m, dtype=torch.float64, device="cuda")
        out = torch.empty(2 * j + 3, dtype=torch.float64, device="cuda")
        coef = torch.empty(2 * j + 2, dtype=torch.float64, device="cuda")
        ws, wsb = runtime.workspace(j + 2)
        st = runtime.stream_handle()
        w2 = torch.empty_like(w)
        t_gram = bench(lambda: _lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(),
                                         aw.data_ptr(), out.data_ptr(), coef.data_ptr(), None, 0,
                                         None, ws, wsb, st))
        t_upd = bench(lambda: _lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(),
                                        w2.data_ptr(), aw.data_ptr(), coef.data_ptr(), 1, None, st))
        print(json.dumps({"m": m, "j": j, "gram_us": round(t_gram, 2), "update_us": round(t_upd, 2),
                          "env": {k: os.environ.get(k) for k in ("KLS_GRAM", "KLS_UPDATE")}}), flush=True)
