"""The row-sharded (N > 1) host logic on CPU with the gloo backend, world
size 2, 3 and 8 (the driver's largest run): the segment row partition, the
CSR halo exchange plan, the one reduction per DCGS2 step through the fixed
segment tree (local tree, exported nodes, combine), and the replicated host
step math -- driving numpy stand-ins for the device kernels (test
scaffolding only) -- reproduce the oracle's Hessenberg matrix and reduction
count, and the one-rank run BITWISE."""

import math
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


def _fdot(a, b):
    """Stand-in for a kernel's fixed-order segment sum (exact-rounded, so the
    same value for the same rows whatever the array's address)."""
    return math.fsum(np.asarray(a) * np.asarray(b))


def _expand(world, rank, k, steps, gather, exchange):
    """The sharded DCGS2 expansion on this rank with numpy stand-ins for the
    kernels.  Reductions follow the device's rank-count-independent scheme:
    per-segment values over the 24 global segments, the rank's local tree
    (seg_local_nodes), an all_gather of the exported nodes and the fixed
    tree's combine (seg_combine_host)."""
    from paper_2104_01253_b200.arnoldi import dcgs2_host_step
    from paper_2104_01253_b200.ledger import MV_TRANS_MV, SyncLedger
    from paper_2104_01253_b200.problems import ManteuffelSpec, halo_plan, manteuffel_build
    from paper_2104_01253_b200.runtime import (seg_combine_host, seg_first, seg_local_nodes,
                                               seg_range, seg_row)

    csr = manteuffel_build(ManteuffelSpec(k=k))
    m = csr.nrows
    lo, hi = seg_range(m, 64, world, rank)
    s, e = csr.indptr[lo], csr.indptr[hi]
    cols = csr.indices[s:e]
    need_lo, need_hi = min(int(cols.min()), lo), max(int(cols.max()) + 1, hi)
    plan = halo_plan(rank, gather([need_lo, lo, hi, need_hi])) if world > 1 else ([], [])
    ptr = csr.indptr[lo : hi + 1] - s
    lcols = cols - need_lo
    vals = csr.data[s:e]
    segs = [(seg_row(m, 64, g) - lo, seg_row(m, 64, g + 1) - lo)
            for g in range(seg_first(rank, world), seg_first(rank + 1, world))]

    def apply(xl):
        ext = np.zeros(need_hi - need_lo)
        ext[lo - need_lo : hi - need_lo] = xl
        lo_buf = np.zeros(lo - need_lo)
        hi_buf = np.zeros(need_hi - hi)
        if world > 1:
            exchange(plan, xl, lo_buf, hi_buf)
        ext[: lo - need_lo] = lo_buf
        ext[hi - need_lo :] = hi_buf
        return oracle.csr_matvec(ptr, lcols, vals, ext)

    def reduce(segval):
        """segval(a, b) -> the values of local rows [a, b); combined."""
        nodes = seg_local_nodes([segval(a, b) for a, b in segs], rank, world)
        blocks = gather(nodes) if world > 1 else [nodes]
        return seg_combine_host(blocks, world)

    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(m)
    led = SyncLedger()
    cap = steps + 1
    Q = np.zeros((hi - lo, cap))
    H = np.zeros((cap, cap - 1))
    w = start[lo:hi].copy()
    wscale = float(np.sqrt(reduce(lambda a, b: np.array([_fdot(w[a:b], w[a:b])]))[0]))
    aw = apply(w)
    K = None
    nb = 0
    for _ in range(steps):
        j = nb

        def gram(a, b):
            q, ws, aws = Q[a:b, :j], w[a:b], aw[a:b]
            return np.array([*(_fdot(q[:, c], ws) for c in range(j)), _fdot(ws, ws),
                             *(_fdot(q[:, c], aws) for c in range(j)), _fdot(ws, aws),
                             _fdot(aws, aws)])

        g = reduce(gram)  # the one global reduction of the step
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
    return H[:nb, : nb - 1].copy(), led.reductions


def _worker(rank, world, port, k, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def gather(obj):
            got = [None] * world
            dist.all_gather_object(got, obj)
            return got

        H, reductions = _expand(world, rank, k, steps, gather, _exchange)
        out[rank] = (H, reductions, world)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_dcgs2_matches_oracle(world):
    """Sharded over gloo ranks, the expansion reproduces the oracle and --
    through the fixed segment tree -- is BITWISE the one-rank run."""
    k, steps = 40, 16
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), k, steps, out), nprocs=world, join=True)
    H1, red1 = _expand(1, 0, k, steps, None, None)
    ptr, idx, dat = oracle.manteuffel_csr(k, 0.5)
    start = np.random.Generator(np.random.PCG64(1729)).standard_normal(k * k)
    exp = oracle.kls_oracle.Dcgs2Expansion(lambda x: oracle.csr_matvec(ptr, idx, dat, x), start,
                                           steps + 1)
    for _ in range(steps):
        exp.step()
    Href = exp.H[: exp.nb, : exp.hcols]
    assert np.max(np.abs(H1 - Href)) <= 1e-12 * np.max(np.abs(Href))
    for r in range(world):
        H, reductions, nranks = out[r]
        assert nranks == world
        assert H.shape == Href.shape
        assert np.array_equal(H, H1)  # rank-count independent
        assert reductions == exp.cnt.reductions == red1


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


def test_segment_partition():
    """Rank row blocks are unions of the 24 global segments: contiguous,
    covering, nearly equal for N | 24, and identical to the library's."""
    from paper_2104_01253_b200.runtime import seg_range

    for n in (0, 1, 7, 100, 10_004_569, 130023424):
        for unit in (64, 262144):
            for parts in (1, 2, 3, 4, 6, 8):
                spans = [seg_range(n, unit, parts, i) for i in range(parts)]
                assert spans[0][0] == 0 and spans[-1][1] == n
                assert all(spans[i][1] == spans[i + 1][0] for i in range(parts - 1))
                assert all(a % unit == 0 for a, _ in spans)
                if n >= 24 * unit * 8:
                    sizes = [b - a for a, b in spans]
                    assert max(sizes) - min(sizes) <= unit * (24 // parts)


def test_segment_tree_exports_and_combine():
    """Every rank split exports a partition of the leaves into maximal
    subtrees (one node per rank when N divides 8), and combining them gives
    the same bits as the one-rank tree."""
    from paper_2104_01253_b200.runtime import (seg_combine_host, seg_exports, seg_first,
                                               seg_local_nodes)

    rng = np.random.default_rng(3)
    leaves = rng.standard_normal((24, 5)) * 10.0 ** rng.integers(-8, 8, size=(24, 1))
    root1 = seg_combine_host([seg_local_nodes(leaves, 0, 1)], 1)
    for world in (1, 2, 3, 4, 5, 6, 7, 8):
        blocks = []
        for r in range(world):
            ids = seg_exports(r, world)
            assert 1 <= len(ids) <= 8
            if 8 % world == 0:
                assert len(ids) == 1
            a, b = seg_first(r, world), seg_first(r + 1, world)
            blocks.append(seg_local_nodes(leaves[a:b], r, world))
        assert np.array_equal(seg_combine_host(blocks, world), root1)


def test_library_segment_layout_matches_host():
    """kls_seg_rows / kls_seg_exports (host functions of the C-ABI, no GPU)
    agree with the Python restatement."""
    import ctypes

    from paper_2104_01253_b200 import _lib
    from paper_2104_01253_b200.runtime import seg_exports, seg_range

    lib = _lib.load()
    for m, unit in ((130023424, 262144), (10_004_569, 64), (777, 64), (5, 64)):
        for world in (1, 2, 3, 4, 8):
            for r in range(world):
                s = _lib.KlsSegs(m, unit, world, r)
                lo, hi = ctypes.c_int64(), ctypes.c_int64()
                assert lib.kls_seg_rows(ctypes.byref(s), ctypes.byref(lo), ctypes.byref(hi)) == 0
                assert (lo.value, hi.value) == seg_range(m, unit, world, r)
                ids = (ctypes.c_int32 * 8)()
                n = lib.kls_seg_exports(r, world, ids)
                assert list(ids[:n]) == seg_exports(r, world)


def _comm_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2104_01253_b200.runtime import Comm

        c = Comm()
        t = torch.full((3,), float(rank + 1), dtype=torch.float64)
        c.allreduce_(t)
        out[rank] = (c.rank, c.world, t.tolist(), c.allreduce_calls,
                     c.allreduce_max_int(rank), c.segs(1000).world)
    finally:
        dist.destroy_process_group()


def test_comm_collectives_gloo():
    """runtime.Comm's own methods on gloo ranks (the NCCL fallback paths of
    the reductions call allreduce_ / combine_ / allreduce_host)."""
    from paper_2104_01253_b200.runtime import Comm

    for name in ("allreduce_", "combine_", "allreduce_host", "allreduce_max_int", "segs", "barrier"):
        assert callable(getattr(Comm, name, None)), name
    world = 3
    out = mp.Manager().dict()
    mp.spawn(_comm_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        rank, w, t, calls, mx, sw = out[r]
        assert (rank, w, calls, mx, sw) == (r, world, 1, world - 1, world)
        assert t == [6.0, 6.0, 6.0]
