"""A/B of the K1 Gram kernel: the current library against the round-1 build
(scripts/exp/libklsgpu_r1.so, rank-order partial sums) at config 3's m.

    python scripts/exp/k1_ab.py [--lib new|r1] [--j 50] [--reps 5]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="new")
    ap.add_argument("--m", type=int, default=130023424)
    ap.add_argument("--j", default="10,50,100")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    from paper_2104_01253_b200 import runtime

    m = a.m
    js = [int(v) for v in a.j.split(",")]
    ld = runtime.pad_rows(m)
    Q = torch.randn((max(js) + 1, ld), dtype=torch.float64, device="cuda")
    w = torch.randn(ld, dtype=torch.float64, device="cuda")
    aw = torch.randn(ld, dtype=torch.float64, device="cuda")
    out = torch.empty(2 * max(js) + 8, dtype=torch.float64, device="cuda")
    ws_t = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    P = ctypes.c_void_p
    if a.lib == "r1":
        lib = ctypes.CDLL(os.path.join(ROOT, "scripts", "exp", "libklsgpu_r1.so"))
        f = lib.kls_gram_dcgs2
        f.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P, P, P, P, ctypes.c_size_t, P]
        call = lambda j: f(Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(), out.data_ptr(),  # noqa: E731
                           ws_t.data_ptr(), ws_t.numel(), st)
    else:
        from paper_2104_01253_b200 import _lib

        lib = _lib.load()
        f = lib.kls_gram_dcgs2
        call = lambda j: f(Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(), out.data_ptr(),  # noqa: E731
                           None, ws_t.data_ptr(), ws_t.numel(), st)
    res = {"lib": a.lib, "m": m, "virt": os.environ.get("KLS_TMA_VIRT", "default")}
    for j in js:
        assert call(j) == 0
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
        for r in range(a.reps):
            ev[2 * r].record()
            call(j)
            ev[2 * r + 1].record()
        torch.cuda.synchronize()
        t = sorted(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(a.reps))[a.reps // 2]
        res[f"j{j}_ms"] = round(t, 4)
        res[f"j{j}_TBs"] = round(8 * m * (j + 2) / t / 1e9, 3)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
