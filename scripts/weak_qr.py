"""Config 5: DCGS2 QR weak-scaling sweep — m = 2.5e7 rows per GPU of a
seeded random-sparse tall-skinny matrix (density 1e-3, N(0,1) values,
generated on each rank's device), n = 25..200 columns, one fused reduction
per column.

    torchrun --nproc-per-node N scripts/weak_qr.py [--m-per-gpu 25000000] [--n 25,50,100,200]

Rank 0 prints one JSON line per n: columns/s for the whole job, the
algorithmic HBM rate per GPU (8 m (2j+6) bytes per column), the loss of
orthogonality, and the reduction count.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m-per-gpu", type=int, default=25_000_000)
    ap.add_argument("--n", default="25,50,100,200")
    ap.add_argument("--density", type=float, default=1e-3)
    a = ap.parse_args()
    from paper_2104_01253_b200 import runtime

    comm = runtime.init_distributed()
    world, rank = comm.world, comm.rank
    import paper_2104_01253_b200 as kls

    m = a.m_per_gpu * world
    lo, hi = runtime.seg_range(m, runtime.row_unit(m), world, rank)  # this rank's rows (24-segment layout)
    ml = hi - lo
    for n in (int(v) for v in a.n.split(",")):
        g = torch.Generator(device="cuda")
        g.manual_seed(1729 + 7919 * rank)
        A = torch.randn((n, ml), generator=g, dtype=torch.float64, device="cuda")
        A *= torch.rand((n, ml), generator=g, device="cuda") < a.density

        def run(led=None):
            st = kls.make_state("dcgs2", m, n, ledger=led)
            for c in range(n):
                st.push(A[c])
            return st.finalize()

        run()
        torch.cuda.synchronize()
        if world > 1:
            comm.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        led = kls.SyncLedger()
        e0.record()
        Q, R = run(led)
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) * 1e-3
        if world > 1:
            sec = comm.allreduce_max_float(sec)
            comm.barrier()
        loo = kls.loss_of_orthogonality(Q, segs=comm.segs(m))
        bytes_per_gpu = sum(8 * (m / world) * (2 * j + 6) for j in range(n))
        if rank == 0:
            print(json.dumps({"config": 5, "gpus": world, "m_per_gpu": ml, "m": m, "n": n,
                              "seconds": sec, "columns_per_s": n / sec,
                              "hbm_GBs_per_gpu": bytes_per_gpu / sec / 1e9, "loo": loo,
                              "reductions": led.reductions}), flush=True)
        del A, Q, R
        torch.cuda.empty_cache()
    runtime.shutdown_distributed()


if __name__ == "__main__":
    main()
