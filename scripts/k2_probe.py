"""Run K2 (kls_dcgs2_update_dev) alone at one size for an ncu capture:

    M=130023424 J=50 python scripts/k2_probe.py
    ncu --set full -k regex:dcgs2_update --launch-skip 2 --launch-count 1 python scripts/k2_probe.py
"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_01253_b200 import _lib, runtime

m, j = int(float(os.environ.get("M", "130023424"))), int(os.environ.get("J", "50"))
ld = runtime.pad_rows(m)
Q = torch.empty((j + 1, ld), dtype=torch.float64, device="cuda")
Q.normal_()
w = torch.randn(m, dtype=torch.float64, device="cuda")
aw = torch.randn(m, dtype=torch.float64, device="cuda")
w2 = torch.empty_like(w)
c = torch.rand(2 * j + 2, dtype=torch.float64, device="cuda") * 0.1 + 1.0
st = runtime.stream_handle()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(6):
    if it == 3:
        e0.record()
    _lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(), w2.data_ptr(),
              aw.data_ptr(), c.data_ptr(), 1, None, st)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 3
print({"m": m, "j": j, "k2_us": round(us, 1), "TBs": round(8 * m * (j + 4) / us / 1e6, 3)})
