"""Host time of one kls_dcgs2_queue_step call (3 launches + event record) at
config 1's size against the device time of the queued chain."""
import ctypes, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2104_01253_b200 as kls
from paper_2104_01253_b200 import _lib as lib, runtime as rt

op = kls.CsrOperator(kls.manteuffel_build(kls.ManteuffelSpec(k=100, beta=0.0)))
m = op.n
ld = rt.pad_rows(m)
J = 52
Q = torch.randn((J + 2, ld), dtype=torch.float64, device="cuda") / np.sqrt(m)
w = torch.randn(m, dtype=torch.float64, device="cuda")
aw = op.apply(w)
w2, a2 = torch.empty_like(w), torch.empty_like(w)
st = rt.stream_handle()
ws, wsb = rt.workspace_for(st, J + 3, m)
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
L = lib.load()
f = L.kls_dcgs2_queue_step
lib.call("kls_gram_dcgs2_step", Q.data_ptr(), ld, m, 25, w.data_ptr(), aw.data_ptr(), gdev.data_ptr(),
         cdev.data_ptr(), gout.data_ptr(), 0, op.segs.ptr, ws, wsb, st)
for _ in range(20):
    f(ctypes.byref(plan), 25, w.data_ptr(), w2.data_ptr(), w2.data_ptr(), aw.data_ptr(), a2.data_ptr(), 0, 1)
torch.cuda.synchronize()
N = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(N):
    f(ctypes.byref(plan), 25, w.data_ptr(), w2.data_ptr(), w2.data_ptr(), aw.data_ptr(), a2.data_ptr(), 0, 1)
t1 = time.perf_counter()
e1.record(); torch.cuda.synchronize()
# the device alone: hold the stream with a sleep kernel while the host
# queues the steps, then time them from an event recorded after the sleep
torch.cuda._sleep(int(2e9 * (N * 20e-6 + 5e-3)))
e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e2.record()
for _ in range(N):
    f(ctypes.byref(plan), 25, w.data_ptr(), w2.data_ptr(), w2.data_ptr(), aw.data_ptr(), a2.data_ptr(), 0, 1)
e3.record(); torch.cuda.synchronize()
print(json.dumps({"m": m, "host_us_per_step": round((t1 - t0) / N * 1e6, 2),
                  "device_us_per_step_host_paced": round(e0.elapsed_time(e1) * 1e3 / N, 2),
                  "device_us_per_step_prequeued": round(e2.elapsed_time(e3) * 1e3 / N, 2)}))
