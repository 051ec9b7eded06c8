"""Fused DCGS2 step (kls_dcgs2_fused_step) vs the three unfused launches at
one step j, device time per step from CUDA events (20 reps after warm-up).
    python scripts/exp/fused_probe.py [k_manteuffel] [j ...]"""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
from paper_2104_01253_b200 import _lib as lib, problems, runtime as rt

kman = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
js = [int(v) for v in sys.argv[2:]] or [10, 25, 50]
op = problems.manteuffel_operator(kls.ManteuffelSpec(k=kman, beta=0.5))
m = op.n
ld = rt.pad_rows(m)
jmax = max(js)
Q = torch.randn((jmax + 2, ld), dtype=torch.float64, device="cuda") / np.sqrt(m)
w = torch.randn(m, dtype=torch.float64, device="cuda")
aw = op.apply(w)
st = rt.stream_handle()
ws, wsb = rt.workspace_for(st, jmax + 3, m)
segp = op.segs.ptr
n = 2 * (jmax + 2) + 3
gdev, cdev, gout = (torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(3))
w1, a1 = torch.empty_like(w), torch.empty_like(w)
ecol, evals, elen, width, eld = op._ell
plan = lib.KlsStepPlan()
plan.Q, plan.ldq, plan.m = Q.data_ptr(), ld, m
plan.segs = op.segs.c
plan.gdev, plan.cdev = gdev.data_ptr(), cdev.data_ptr()
plan.gout[0] = plan.gout[1] = gout.data_ptr()
plan.ws, plan.ws_bytes, plan.stream = ws, wsb, st
plan.divide, plan.qr = 1, 0
plan.op = op.op_desc()


def coef(j):
    lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
             gdev.data_ptr(), cdev.data_ptr(), gout.data_ptr(), 0, segp, ws, wsb, st)


def unfused(j):
    lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(), w1.data_ptr(),
             aw.data_ptr(), cdev.data_ptr(), 1, segp, st)
    lib.call("kls_ell_spmv", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(), width, m, eld,
             w1.data_ptr(), a1.data_ptr(), st)
    lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j + 1, w1.data_ptr(), a1.data_ptr(),
             gdev.data_ptr(), cdev.data_ptr(), gout.data_ptr(), 0, segp, ws, wsb, st)


def fused(j):
    lib.call("kls_dcgs2_fused_step", ctypes.byref(plan), j, w.data_ptr(), w1.data_ptr(),
             aw.data_ptr(), a1.data_ptr(), 0)


def timeit(fn, j, reps=20):
    for _ in range(3):
        coef(j); fn(j)
    ts = []
    for _ in range(reps):
        coef(j)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(j); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def traced(j):
    nit = (m + 1023) // 1024 + 24
    tr = torch.zeros(8 * nit, dtype=torch.int64, device="cuda")
    coef(j)
    lib.call("kls_dcgs2_fused_step_traced", ctypes.byref(plan), j, w.data_ptr(), w1.data_ptr(),
             aw.data_ptr(), a1.data_ptr(), 0, tr.data_ptr())
    torch.cuda.synchronize()
    t = tr.view(-1, 8).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    it_us = (t[148:, 6] - t[:-148, 6]) / 1e3 if len(t) > 148 else np.zeros(1)
    med = lambda a: round(float(np.median(a)), 2)
    return {"items": len(t), "span_us": round(float((t[:, 6].max() - t0) / 1e3), 1),
            "iter_us": med(it_us), "U_throttle_us": med((t[:, 1] - t[:, 0]) / 1e3),
            "U_us": med((t[:, 2] - t[:, 1]) / 1e3),
            "G_halo_wait_us": med((t[:, 4] - t[:, 3]) / 1e3),
            "G_start_minus_U_pub_us": med((t[:, 3] - t[:, 2]) / 1e3),
            "K3_us": med((t[:, 5] - t[:, 4]) / 1e3), "K1_us": med((t[:, 6] - t[:, 5]) / 1e3)}


out = {"m": m, "hint": os.environ.get("KLS_FUSED_HINT", "1")}
elig = lib.load().kls_dcgs2_fused_eligible(ctypes.byref(plan), js[0]) == 1
out["tree"] = "chunk" if elig else "items"
for j in js:
    tu = timeit(unfused, j)
    tf = timeit(fused, j) if elig else float("nan")
    b = 8 * m * (2 * j + 8) + 61 * m  # unfused algorithmic bytes
    if elig:
        out[f"trace_j{j}"] = traced(j)
    out[f"j{j}"] = {"unfused_us": round(tu, 1), "fused_us": round(tf, 1),
                    "unfused_GBs": round(b / tu / 1e3), "fused_eff_GBs": round(b / tf / 1e3) if elig else None}
print(json.dumps(out))
