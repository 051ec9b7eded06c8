"""Micro-benchmark: kls_project_gram (CGS2's fused update + projection) vs a
plain projection (kls_mv_trans_mv) over the same Q panel.

    python scripts/pg_bench.py [--m 130023424] [--k 25,50,100] [--reps 5]

Prints one JSON line per k: ms per call and the algorithmic GB/s of each
(project: 8m(k+1); project_gram: 8m(k+2)).
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=130_023_424)
    ap.add_argument("--k", default="25,50,100")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from paper_2104_01253_b200 import _lib, runtime

    ks = [int(v) for v in a.k.split(",")]
    kmax = max(ks)
    m = a.m
    ld = runtime.pad_rows(m)
    Q = torch.randn((kmax, ld), dtype=torch.float64, device="cuda")
    v = torch.randn(ld, dtype=torch.float64, device="cuda")
    out = torch.empty(kmax + 2, dtype=torch.float64, device="cuda")
    ws, wsb = runtime.workspace(kmax + 2)
    st = runtime.stream_handle()
    stream = torch.cuda.current_stream()
    for k in ks:
        s = np.random.default_rng(k).standard_normal(k) * 1e-3
        res = {}
        for name in ("project", "project_gram"):
            def call():
                if name == "project":
                    _lib.call("kls_mv_trans_mv", Q.data_ptr(), ld, m, k, None, v.data_ptr(), None, 1,
                              1, out.data_ptr(), None, ws, wsb, st)
                else:
                    _lib.call("kls_project_gram", Q.data_ptr(), ld, m, k, v.data_ptr(),
                              s.ctypes.data, 1, 1, out.data_ptr(), None, ws, wsb, st)
            for _ in range(2):
                call()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.reps):
                call()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            nb = 8 * m * (k + (1 if name == "project" else 2))
            res[name] = {"ms": ms, "gbs": nb / ms / 1e6}
        print(json.dumps({"m": m, "k": k, **res}), flush=True)


if __name__ == "__main__":
    main()
