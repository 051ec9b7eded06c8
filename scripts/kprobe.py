"""Kernel probe: time the K1 Gram, K2 update and K3 operator kernels at a
large m with CUDA events and print achieved HBM GB/s per kernel.

    python scripts/kprobe.py [--m 130023424] [--j 10,50,100] [--reps 5]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2104_01253_b200 import _lib, laplace3d, runtime  # noqa: E402


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for r in range(reps):
        ev[2 * r].record()
        fn()
        ev[2 * r + 1].record()
    torch.cuda.synchronize()
    t = sorted(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps))
    return t[len(t) // 2] * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="496,512,512")
    ap.add_argument("--j", default="10,50,100")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dims = tuple(int(v) for v in a.dims.split(","))
    m = dims[0] * dims[1] * dims[2]
    js = [int(v) for v in a.j.split(",")]
    jmax = max(js)
    ld = runtime.pad_rows(m)
    lib = _lib.load()
    Q = torch.randn((jmax + 1, ld), dtype=torch.float64, device="cuda")
    w = torch.randn(ld, dtype=torch.float64, device="cuda")[:m]
    aw = torch.randn(ld, dtype=torch.float64, device="cuda")[:m]
    out = torch.empty(2 * jmax + 8, dtype=torch.float64, device="cuda")
    ws, wsb = runtime.workspace(jmax + 1)
    st = runtime.stream_handle()
    res = {"m": m, "sm": lib.kls_device_sm_count()}
    for j in js:
        coef = torch.randn(2 * j + 1, dtype=torch.float64, device="cuda") * 1e-3
        g = timeit(lambda: _lib.call("kls_gram_dcgs2", Q.data_ptr(), ld, m, j, w.data_ptr(),
                                     aw.data_ptr(), out.data_ptr(), None, ws, wsb, st), a.reps)
        u = timeit(lambda: _lib.call("kls_dcgs2_update", Q.data_ptr(), ld, m, j, w.data_ptr(),
                                     aw.data_ptr(), coef.data_ptr(), 1.0, 1, None, st), a.reps)
        res[f"gram_j{j}_ms"] = g * 1e3
        res[f"gram_j{j}_GBs"] = 8 * m * (j + 2) / g / 1e9
        res[f"update_j{j}_ms"] = u * 1e3
        res[f"update_j{j}_GBs"] = 8 * m * (j + 4) / u / 1e9
    op = laplace3d(*dims)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    s = timeit(lambda: op.apply_into(w, y), a.reps)
    res["stencil_ms"] = s * 1e3
    res["stencil_GBs"] = 16 * m / s / 1e9
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
