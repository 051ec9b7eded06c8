"""Time the step's Gram -> update kernel pair back to back (CUDA events), to
see what launching the update as a programmatic dependent (PDL) saves.

    SIZES=1e4,1e6 python scripts/chain_probe.py      # KLS_PDL=0 for plain launches
"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_01253_b200 import _lib, runtime

for m in [int(float(v)) for v in os.environ.get("SIZES", "1e4,1e5,1e6,1e7").split(",")]:
    for j in (25, 50):
        ld = runtime.pad_rows(m)
        Q = torch.randn((j + 1, ld), dtype=torch.float64, device="cuda") / np.sqrt(m)
        w = torch.randn(m, dtype=torch.float64, device="cuda")
        aw = torch.randn(m, dtype=torch.float64, device="cuda")
        w2 = torch.empty_like(w)
        g = torch.empty(2 * j + 3, dtype=torch.float64, device="cuda")
        c = torch.empty(2 * j + 2, dtype=torch.float64, device="cuda")
        ws, wsb = runtime.workspace(j + 2)
        st = runtime.stream_handle()

        def pair():
            _lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
                      g.data_ptr(), c.data_ptr(), None, 0, None, ws, wsb, st)
            _lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(), w2.data_ptr(),
                      aw.data_ptr(), c.data_ptr(), 1, None, st)

        for _ in range(5):
            pair()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 100
        e0.record()
        for _ in range(reps):
            pair()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"m": m, "j": j, "pair_us": round(e0.elapsed_time(e1) * 1e3 / reps, 2),
                          "pdl": os.environ.get("KLS_PDL", "1")}), flush=True)
