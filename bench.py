#!/usr/bin/env python
"""bench.py — DCGS2 Arnoldi-QR throughput on B200 (BASELINE.json config 3).

Workload: ``arnoldi_expand(laplace3d(496, 512, 512), start, "dcgs2", 100)``,
m = 130,023,424 rows, n = 100 Krylov vectors, fp64, matrix-free 7-point
operator; Q (105 GB) never fits the 126 MB L2.  One bench "step" is one full
expansion (100 Arnoldi iterations plus the finalize flush).  Rows are
sharded over the ranks (strong scaling: the same m at every N).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

``value`` = Arnoldi iterations/s with the start vector resident in HBM;
``e2e`` = the same through the public API from a pinned host start vector
(H2D inside the timed region, the per-iteration scalars D2H).  Rank 0 prints
one JSON line.  ``--impl reference`` times the reference's own CPU
implementation (kls from baseline/_ref, else the oracle port) on the host
cores over a bounded sample of the workload (fewer rows, same n), scaled to
the full m by row count (all terms are linear in m).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DCGS2 Arnoldi iters/sec + HBM GB/s (fp64) at 1/2/4/8 B200 vs CPU ref"
UNIT = "iters/s"
FULL_DIMS = (496, 512, 512)
SAMPLE_DIMS = (31, 64, 128)  # 1/512 of the rows: ~5 s per expansion on 8 cores
NOMINAL_HBM_GBS = 8000.0
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--dims", default=",".join(map(str, FULL_DIMS)))
    ap.add_argument("--n", type=int, default=100, help="Arnoldi iterations per expansion")
    ap.add_argument("--scheme", default="dcgs2", choices=("dcgs2", "cgs2"))
    ap.add_argument("--operator", default="stencil", choices=("stencil", "csr"),
                    help="matrix-free stencil (the reference's laplace3d) or the same "
                         "operator as a device-assembled CSR matrix")
    ap.add_argument("--sample-dims", default=",".join(map(str, SAMPLE_DIMS)))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dims_of(s):
    return tuple(int(v) for v in s.split(","))


def workload_name(dims, n, scheme, operator="stencil"):
    m = dims[0] * dims[1] * dims[2]
    form = "matrix-free 7-point" if operator == "stencil" else "7-point as CSR"
    return f"{scheme} Arnoldi-QR, laplace3d{dims} {form}, m={m}, n={n}"


# ---------------------------------------------------------------------------
# CPU side: the reference implementation (or the oracle port) on host cores


def cpu_reference_rate(sample_dims, n, scheme, reps=1):
    """(iters/s at the sample size, kind, seconds per expansion)."""
    import numpy as np

    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    kind = "port"
    try:
        if os.path.isdir(os.path.join(ref_dir, "kls")):
            sys.path.insert(0, ref_dir)
            import kls  # the unmodified reference (pip-installed into baseline/_ref)

            kind = "reference"
    except Exception:
        kind = "port"
    m = sample_dims[0] * sample_dims[1] * sample_dims[2]
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(m)
    times = []
    for _ in range(reps):
        if kind == "reference":
            op = kls.laplace3d(*sample_dims)
            t0 = time.perf_counter()
            kls.arnoldi_expand(op, start, scheme, n)
            times.append(time.perf_counter() - t0)
        else:
            import oracle  # CPU restatement (test infrastructure), baseline leg only

            fn = getattr(oracle, f"{scheme}_arnoldi")
            t0 = time.perf_counter()
            fn(lambda x: oracle.stencil7_matvec(x, sample_dims), start, n)
            times.append(time.perf_counter() - t0)
    return n / statistics.median(times), kind, times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    dims = dims_of(args.dims)
    sdims = dims_of(args.sample_dims)
    m, ms = dims[0] * dims[1] * dims[2], sdims[0] * sdims[1] * sdims[2]
    for _ in range(args.warmup):
        cpu_reference_rate(sdims, args.n, args.scheme)
    rate, kind, times = cpu_reference_rate(sdims, args.n, args.scheme, reps=max(args.steps, 1))
    value = rate * ms / m
    cores = os.cpu_count()
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.median(times) * m / ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: PCG64(1729) standard-normal start vector",
        "config": {"workload": workload_name(dims, args.n, args.scheme, args.operator), "m": m, "n": args.n,
                   "sample_rows": ms, "sample_dims": list(sdims),
                   "extrapolation": "iters/s at the sample size x (sample rows / m)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"{args.scheme} arnoldi_expand n={args.n} on laplace3d{sdims} "
                                   f"({ms} rows), {len(times)} timed runs, OpenBLAS default threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.idx)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            p = [v.strip() for v in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU side


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full
    summary (profiles/ncu_summary.json), with the launch's algorithmic bytes."""
    for name in ("ncu_summary.json", "ncu_summary_cgs2.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                d = json.load(f)
        except Exception:
            continue
        if d.get(kernel):
            return d[kernel]
    return None


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2104_01253_b200 as kls
    from paper_2104_01253_b200 import _lib, runtime, trace

    dims = dims_of(args.dims)
    m = dims[0] * dims[1] * dims[2]
    op = kls.laplace3d(*dims) if args.operator == "stencil" else kls.laplace3d_csr_operator(*dims)
    lo, hi = op.row_lo, op.row_hi
    # start vector: the global PCG64(1729) stream, this rank's rows
    full = np.random.Generator(np.random.PCG64(1729)).standard_normal(m)
    start_host = torch.from_numpy(full).pin_memory()
    del full
    start_dev = start_host[lo:hi].to(torch.device("cuda", local))
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        return float(t.item())

    def expansion(start):
        V, H = kls.arnoldi_expand(op, start, args.scheme, args.n)
        return H

    for _ in range(args.warmup):
        expansion(start_dev)
    torch.cuda.synchronize()
    barrier()

    # ---- value: start resident in HBM -------------------------------------
    rec = trace.start(events=True)
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            H = expansion(start_dev)
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    trace.stop()
    launches = _lib.launch_count() - launches0
    sec = max_over_ranks(ev0.elapsed_time(ev1) * 1e-3)
    iters = args.steps * args.n
    value = iters / sec
    # per-kernel device time is read from the recorder spans below
    ar_s, halo_s = rec.seconds("allreduce"), rec.seconds("halo")
    local_bytes = rec.total_bytes()
    total_bytes = sum_over_ranks(local_bytes)
    total_launches = int(sum_over_ranks(launches))

    # ---- e2e: pinned host start, H2D inside the timed region ----------------
    e2e = None
    if not args.no_e2e:
        expansion(start_host)  # warm the host path once
        torch.cuda.synchronize()
        x0 = dict(runtime.XFER)
        barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            H = expansion(start_host)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        wall = time.perf_counter() - t0
        esec = max_over_ranks(max(e0.elapsed_time(e1) * 1e-3, wall))
        h2d = (runtime.XFER["h2d"] - x0["h2d"]) / args.steps
        d2h = (runtime.XFER["d2h"] - x0["d2h"]) / args.steps
        e2e = {"value": iters / esec, "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(h2d)),
               "d2h_bytes_per_step": int(sum_over_ranks(d2h)),
               "path": "kls.arnoldi_expand(op, pinned host start) -> (V on device, H on host)"}

    # ---- collective latency (2j+3 = 203 doubles, back to back) ----------------
    coll = None
    if world > 1:
        coll = {}
        n_ar, reps = 2 * args.n + 3, 200
        src = torch.zeros(n_ar, dtype=torch.float64, device="cuda")
        out = torch.zeros(n_ar, dtype=torch.float64, device="cuda")
        link = runtime.peer_link(op.comm)
        st = runtime.stream_handle()
        for name in ("peer", "nccl"):
            if name == "peer" and link is None:
                continue
            for rep in range(2):  # warm-up pass, timed pass
                barrier()
                torch.cuda.synchronize()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record()
                for _ in range(reps):
                    if name == "peer":
                        link.allreduce(src.data_ptr(), n_ar, out.data_ptr(), st)
                    else:
                        dist.all_reduce(src)
                a1.record()
                torch.cuda.synchronize()
            coll[f"{name}_allreduce_us"] = max_over_ranks(a0.elapsed_time(a1) * 1e3 / reps)
        coll["doubles"] = n_ar
        coll["note"] = ("the step's reduction runs fused into K1 (kls_gram_dcgs2_peer); these are "
                        "standalone back-to-back latencies of the same payload")

    # ---- roofline of the dominant kernel -------------------------------------
    peak, peak_src = measured_peak()
    spans = {name: rec.seconds(name) for name in ("gram", "update", "project", "project_gram", "mtm", "apply")}
    kern = max(spans, key=spans.get)
    k_s = spans[kern]
    k_bytes = rec.bytes[kern]
    k_calls = rec.calls[kern]
    achieved = k_bytes / k_s / 1e9
    traffic = ncu_traffic(kern)
    roofline = {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                "frac_of_8TBs": achieved / NOMINAL_HBM_GBS,
                "bytes_per_launch_avg": k_bytes / max(k_calls, 1),
                "launch_ms_avg": 1e3 * k_s / max(k_calls, 1),
                "share_of_step": k_s / (sec * 1.0) if world == 1 else None,
                "traffic": traffic.get("dram_bytes") if traffic else None,
                "traffic_detail": traffic}

    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * sec / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: PCG64(1729) standard-normal start vector, matrix-free 3-D Poisson",
        "config": {"workload": workload_name(dims, args.n, args.scheme, args.operator), "m": m, "n": args.n,
                   "scheme": args.scheme,
                   "operator": ("laplace3d 7-point, matrix-free" if args.operator == "stencil"
                                else "laplace3d 7-point as device-assembled CSR (int32 cols)"),
                   "parallelism": f"row-shard over {world} GPU(s), 1 allreduce/iteration",
                   "l2": "inputs larger than L2 (Q = %.1f GB)" % (8 * m * (args.n + 1) / 1e9)},
        "hbm_gbs": total_bytes / sec / 1e9 / world,
        "hbm_gbs_total": total_bytes / sec / 1e9,
        "hbm_frac_of_8TBs": total_bytes / sec / 1e9 / world / NOMINAL_HBM_GBS,
        "phase_ms_per_iter": {k: 1e3 * v / iters for k, v in spans.items() if v > 0},
        "allreduce_us_per_iter": 1e6 * ar_s / iters if world > 1 else 0.0,
        "collective_latency": coll,
        "halo_us_per_iter": 1e6 * halo_s / iters if world > 1 else 0.0,
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": total_launches,
        "gpu_launches_per_iter_per_rank": launches / iters,
        "clocks": clk.summary(),
        "reductions_per_iter": 1 if args.scheme == "dcgs2" else 3,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sdims = dims_of(args.sample_dims)
        ms = sdims[0] * sdims[1] * sdims[2]
        rate, kind, times = cpu_reference_rate(sdims, args.n, args.scheme)
        line["cpu_baseline"] = {
            "value": rate * ms / m, "unit": UNIT, "cores": os.cpu_count(), "kind": kind,
            "sample": f"{args.scheme} arnoldi_expand n={args.n} on laplace3d{sdims} ({ms} rows, "
                      f"{times[0]:.1f} s), scaled by rows to m={m}; OpenBLAS default threads"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
