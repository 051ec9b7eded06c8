"""Operator-apply probe: time one y = A x of the device-built CSR operators
(ELL copy when rows are short) with CUDA events; print the algorithmic
HBM GB/s (CsrOperator.apply_bytes).

    python scripts/spmv_probe.py [--lap 496,512,512] [--mant 3163] [--reps 5]
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lap", default="496,512,512")
    ap.add_argument("--mant", type=int, default=3163)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import paper_2104_01253_b200 as kls
    from paper_2104_01253_b200 import problems

    ops = []
    if a.lap:
        nx, ny, nz = (int(v) for v in a.lap.split(","))
        ops.append((f"laplace3d_csr{nx}x{ny}x{nz}", lambda: problems.laplace3d_csr_operator(nx, ny, nz)))
    if a.mant:
        ops.append((f"manteuffel{a.mant}", lambda: problems.manteuffel_operator(
            kls.ManteuffelSpec(k=a.mant, beta=0.5))))
    for name, make in ops:
        op = make()
        x = op.new_vector()
        x.local.copy_(torch.randn(op.m_local, dtype=torch.float64, device="cuda"))
        y = torch.empty(op.m_local, dtype=torch.float64, device="cuda")
        for _ in range(2):
            op.apply_into(x, y)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            op.apply_into(x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        nb = op.apply_bytes()
        print(json.dumps({"op": name, "m": op.m_local, "ell": op._ell is not None, "ms": ms,
                          "bytes": nb, "gbs": nb / ms / 1e6}), flush=True)
        del op, x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
