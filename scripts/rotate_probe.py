"""Krylov-Schur rotation kernel (kls_tsgemm_inplace_cols) at config 4's
size: m = 1e7 rows, k = 60 basis columns, p = 30 kept columns; CUDA-event
time and the achieved HBM rate on its 8 m (k + p) algorithmic bytes.  The
default is the DMMA kernel; KLS_ROTATE=fma selects the DFMA one.

    python scripts/rotate_probe.py; KLS_ROTATE=fma python scripts/rotate_probe.py
"""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_01253_b200 import _lib, runtime

m = 10_004_569
ld = runtime.pad_rows(m)
cases = ((60, 30), (60, 60), (30, 15))
if os.environ.get("ROT_CASES"):  # e.g. ROT_CASES=60x30 (ncu captures)
    cases = tuple(tuple(int(v) for v in c.split("x")) for c in os.environ["ROT_CASES"].split(","))
for k, p in cases:
    V = torch.randn((k, ld), dtype=torch.float64, device="cuda")
    Z = torch.randn(k * p, dtype=torch.float64, device="cuda") / k
    st = runtime.stream_handle()
    for _ in range(3):
        _lib.call("kls_tsgemm_inplace_cols", V.data_ptr(), ld, m, k, p, Z.data_ptr(), st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        _lib.call("kls_tsgemm_inplace_cols", V.data_ptr(), ld, m, k, p, Z.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"kernel": os.environ.get("KLS_ROTATE", "mma"), "m": m, "k": k, "p": p,
                      "ms": round(ms, 3),
                      "TBs": round(8 * m * (k + p) / ms / 1e9, 2),
                      "fp64_TFs": round(2 * m * k * p / ms / 1e9, 2)}))
