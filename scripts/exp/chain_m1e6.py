"""Device time per DCGS2 step of the step plan's chain (update -> ELL ->
Gram + scalar step) at config 2's operator (m = 1e6), back to back at a
fixed j, against each kernel alone.  Prints one JSON line."""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
from paper_2104_01253_b200 import _lib as lib, problems, runtime as rt

op = problems.manteuffel_operator(kls.ManteuffelSpec(k=int(os.environ.get("KMAN", 1000)), beta=0.5))
m = op.n
ld = rt.pad_rows(m)
J = 60
Q = torch.randn((J + 2, ld), dtype=torch.float64, device="cuda") / np.sqrt(m)
w = torch.randn(m, dtype=torch.float64, device="cuda")
aw = op.apply(w)
w2, a2 = torch.empty_like(w), torch.empty_like(w)
st = rt.stream_handle()
ws, wsb = rt.workspace_for(st, J + 3, m)
segp = op.segs.ptr
n = 2 * J + 8
gdev, cdev = (torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(2))
gout = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
plan = lib.KlsStepPlan()
plan.Q, plan.ldq, plan.m = Q.data_ptr(), ld, m
plan.segs = op.segs.c
plan.gdev, plan.cdev = gdev.data_ptr(), cdev.data_ptr()
plan.gout[0], plan.gout[1] = gout.data_ptr(), gout.data_ptr() + 8 * n
plan.ws, plan.ws_bytes, plan.stream = ws, wsb, st
evs = []
for _ in range(2):
    ev = ctypes.c_void_p(); lib.call("kls_event_create", ctypes.byref(ev)); evs.append(ev.value)
plan.event[0], plan.event[1] = evs
plan.divide, plan.qr = 1, 0
plan.op = op.op_desc()
ecol, evals, elen, width, eld = op._ell


def coef(j):
    lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
             gdev.data_ptr(), cdev.data_ptr(), gout.data_ptr(), 0, segp, ws, wsb, st)


def timed(fn, reps=20):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


out = {"m": m}
for j in (10, 25, 50):
    coef(j)
    # the real chain: queue_step at the same j (coefficients re-made by the Gram each step)
    chain = timed(lambda: lib.call("kls_dcgs2_queue_step", ctypes.byref(plan), j, w.data_ptr(),
                                   w2.data_ptr(), w2.data_ptr(), aw.data_ptr(), a2.data_ptr(), 0, 1))
    upd = timed(lambda: lib.call("kls_dcgs2_update_dev", Q.data_ptr(), ld, m, j, w.data_ptr(),
                                 w2.data_ptr(), aw.data_ptr(), cdev.data_ptr(), 1, segp, st))
    ell = timed(lambda: lib.call("kls_ell_spmv", ecol.data_ptr(), evals.data_ptr(), elen.data_ptr(),
                                 width, m, eld, w2.data_ptr(), a2.data_ptr(), st))
    gram = timed(lambda: lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, j + 1, w2.data_ptr(),
                                  a2.data_ptr(), gdev.data_ptr(), cdev.data_ptr(), gout.data_ptr(), 0,
                                  segp, ws, wsb, st))
    bytes_ = 8 * m * (j + 4) + 8 * m * (j + 3) + m * (12 * width + 17)
    out[f"j{j}"] = {"chain_us": round(chain, 1), "update_us": round(upd, 1), "ell_us": round(ell, 1),
                    "gram_us": round(gram, 1), "sum_us": round(upd + ell + gram, 1),
                    "ideal_us_at_6.5TBs": round(bytes_ / 6.5e6, 1)}
print(json.dumps(out))
