"""The row-sharded (N > 1) host logic on CPU with the gloo backend, world
size 2, 3 and 8 (the driver's largest run): row partition, the CSR halo
exchange plan, the one allreduce per DCGS2 step, and the replicated host step math — driving numpy stand-ins
for the device kernels (test scaffolding only) — reproduce the oracle's
single-process Hessenberg matrix and reduction count."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(plan, local, lo_buf, hi_buf):
    sends, recvs = plan
    reqs = []
    for q, a, b in sends:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(local[a:b])), q))
    got = []
    for q, side, a, b in recvs:
        t = torch.empty(b - a, dtype=torch.float64)
        reqs.append(dist.irecv(t, q))
        got.append((side, a, b, t))
    for r in reqs:
        r.wait()
    for side, a, b, t in got:
        (lo_buf if side == "lo" else hi_buf)[a:b] = t.numpy()


def _worker(rank, world, port, k, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_01253_b200.arnoldi import dcgs2_host_step
        from paper_2104_01253_b200.ledger import MV_TRANS_MV, SyncLedger
        from paper_2104_01253_b200.problems import ManteuffelSpec, halo_plan, manteuffel_build
        from paper_2104_01253_b200.runtime import block_range

        csr = manteuffel_build(ManteuffelSpec(k=k))
        m = csr.nrows
        lo, hi = block_range(m, world, rank)
        s, e = csr.indptr[lo], csr.indptr[hi]
        cols = csr.indices[s:e]
        need_lo, need_hi = min(int(cols.min()), lo), max(int(cols.max()) + 1, hi)
        win = torch.tensor([need_lo, lo, hi, need_hi], dtype=torch.int64)
        allw = [torch.empty_like(win) for _ in range(world)]
        dist.all_gather(allw, win)
        plan = halo_plan(rank, [tuple(w.tolist()) for w in allw])
        ptr = csr.indptr[lo : hi + 1] - s
        lcols = cols - need_lo
        vals = csr.data[s:e]

        def apply(xl):
            ext = np.zeros(need_hi - need_lo)
            ext[lo - need_lo : hi - need_lo] = xl
            lo_buf = np.zeros(lo - need_lo)
            hi_buf = np.zeros(need_hi - hi)
            _exchange(plan, xl, lo_buf, hi_buf)
            ext[: lo - need_lo] = lo_buf
            ext[hi - need_lo :] = hi_buf
            return oracle.csr_matvec(ptr, lcols, vals, ext)

        def allreduce(v):
            t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        start = np.random.Generator(np.random.PCG64(1729)).standard_normal(m)
        led = SyncLedger()
        cap = steps + 1
        Q = np.zeros((hi - lo, cap))
        H = np.zeros((cap, cap - 1))
        w = start[lo:hi].copy()
        wscale = float(np.sqrt(allreduce([w @ w])[0]))
        aw = apply(w)
        K = None
        nb = 0
        for _ in range(steps):
            j = nb
            g_local = np.concatenate([Q[:, :j].T @ w, [w @ w], Q[:, :j].T @ aw, [w @ aw],
                                      [aw @ aw]])
            g = allreduce(g_local)  # the one global reduction of the step
            led.record(MV_TRANS_MV, 2 * m * (j + 1) * 2)
            res = dcgs2_host_step(g, j, m, wscale, K, H, led)
            assert res is not None
            c, t, alpha, vscale, K = res
            q = (w - Q[:, :j] @ c) / alpha
            Q[:, j] = q
            w = aw / alpha - (Q[:, :j] @ t[:j] + q * t[j])
            nb += 1
            aw = apply(w)
            wscale = vscale
        out[rank] = (H[:nb, : nb - 1].copy(), led.reductions, allreduce([1.0])[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_dcgs2_matches_oracle(world):
    k, steps = 12, 16
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), k, steps, out), nprocs=world, join=True)
    ptr, idx, dat = oracle.manteuffel_csr(k, 0.5)
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(k * k)
    exp = oracle.kls_oracle.Dcgs2Expansion(lambda x: oracle.csr_matvec(ptr, idx, dat, x), start,
                                           steps + 1)
    for _ in range(steps):
        exp.step()
    Href = exp.H[: exp.nb, : exp.hcols]
    for r in range(world):
        H, reductions, nranks = out[r]
        assert nranks == world
        assert H.shape == Href.shape
        assert np.max(np.abs(H - Href)) <= 1e-12 * np.max(np.abs(Href))
        assert reductions == exp.cnt.reductions
    # every rank took identical host decisions
    for r in range(1, world):
        assert np.array_equal(out[r][0], out[0][0])


def test_halo_plan_symmetry():
    from paper_2104_01253_b200.problems import halo_plan

    rng = np.random.default_rng(0)
    for world in (2, 3, 5, 8):
        bounds = np.sort(rng.choice(np.arange(1, 100), size=world - 1, replace=False))
        edges = [0, *bounds.tolist(), 100]
        wins = []
        for q in range(world):
            lo, hi = edges[q], edges[q + 1]
            wins.append((max(0, lo - int(rng.integers(0, 30))), lo, hi,
                         min(100, hi + int(rng.integers(0, 30)))))
        plans = [halo_plan(r, wins) for r in range(world)]
        # every receive is matched by exactly one send of the same length
        for r, (_, recvs) in enumerate(plans):
            for q, side, a, b in recvs:
                sends_q = [(p, x, y) for p, x, y in plans[q][0] if p == r]
                assert len(sends_q) == 1 and sends_q[0][2] - sends_q[0][1] == b - a
        # halos cover exactly the need windows
        for r, (_, recvs) in enumerate(plans):
            nl, lo, hi, nh = wins[r]
            assert sum(b - a for _, s, a, b in recvs if s == "lo") == lo - nl
            assert sum(b - a for _, s, a, b in recvs if s == "hi") == nh - hi


def test_block_range_partition():
    from paper_2104_01253_b200.runtime import block_range

    for n in (0, 1, 7, 100, 130023424):
        for parts in (1, 2, 3, 8):
            spans = [block_range(n, parts, i) for i in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(parts - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
