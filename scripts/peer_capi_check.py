"""Multi-GPU check of the C-ABI peer path without torch's symmetric memory:
every rank allocates its peer buffer with kls_peer_buffer_alloc, the IPC
handles are exchanged (here over torch.distributed objects; a C host would
use MPI or a socket), peers are opened with kls_peer_buffer_open, and the
one-shot segment-tree combine (kls_peer_seg_combine) and the fused Gram +
combine (kls_gram_dcgs2_peer, with its KlsSegs layout) run on that pointer
table; the fused Gram must equal, bit for bit, the same reduction on ONE
rank holding all rows.  Ranks may share a GPU (LOCAL_RANK % device count).
Rank 0 prints one JSON line; exit 1 on a mismatch.

    torchrun --nproc-per-node N scripts/peer_capi_check.py
"""

import ctypes
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2104_01253_b200 import _lib, runtime

    lib = _lib.load()
    cap = 4096
    nbytes = lib.kls_peer_buffer_bytes(cap)
    hbytes = lib.kls_ipc_handle_bytes()
    handle = (ctypes.c_char * hbytes)()
    mine = ctypes.c_void_p()
    _lib.call("kls_peer_buffer_alloc", nbytes, ctypes.byref(mine), handle)
    handles = [None] * world
    dist.all_gather_object(handles, bytes(handle))
    ptrs = []
    for r in range(world):
        if r == rank:
            ptrs.append(mine.value)
        else:
            p = ctypes.c_void_p()
            h = (ctypes.c_char * hbytes).from_buffer_copy(handles[r])
            _lib.call("kls_peer_buffer_open", h, ctypes.byref(p))
            ptrs.append(p.value)
    table = (ctypes.c_void_p * world)(*ptrs)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    st = runtime.stream_handle()
    ok = True
    res = {"world": world}

    # one-shot combine of exported tree nodes, several epochs: equal to the
    # host restatement of the fixed tree (runtime.seg_combine_host) on all ranks
    for epoch in range(1, 6):
        n = 37 * epoch
        rng = np.random.default_rng(1000 * epoch)
        leaves = rng.standard_normal((24, n)) * 10.0 ** rng.integers(-6, 6, size=(24, 1))
        blocks = []
        for r in range(world):
            a, b = runtime.seg_first(r, world), runtime.seg_first(r + 1, world)
            blocks.append(runtime.seg_local_nodes(leaves[a:b], r, world))
        src = torch.from_numpy(np.ascontiguousarray(blocks[rank])).cuda()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("kls_peer_seg_combine", src.data_ptr(), n, out.data_ptr(), table, rank, world,
                  cap, epoch, err.data_ptr(), st)
        torch.cuda.synchronize()
        want = runtime.seg_combine_host(blocks, world)
        ok = ok and np.array_equal(out.cpu().numpy(), want) and int(err.item()) == 0
    res["combine_ok"] = ok

    # fused Gram + combine over a row-sharded basis, bitwise equal to one
    # rank holding all rows (the same KlsSegs layout at world 1)
    m, j = 400_037, 9
    g = np.random.default_rng(7)
    Q = g.standard_normal((m, j))
    w = g.standard_normal(m)
    aw = g.standard_normal(m)

    def gram(lo, hi, segs, peer):
        ml = hi - lo
        ld = runtime.pad_rows(ml)
        qb = torch.zeros((j, ld), dtype=torch.float64, device="cuda")
        qb[:, :ml] = torch.from_numpy(np.ascontiguousarray(Q[lo:hi].T)).cuda()
        wd = torch.from_numpy(w[lo:hi].copy()).cuda()
        awd = torch.from_numpy(aw[lo:hi].copy()).cuda()
        out = torch.empty(2 * j + 3, dtype=torch.float64, device="cuda")
        ws, wsb = runtime.workspace(j + 2)
        if peer:
            _lib.call("kls_gram_dcgs2_peer", qb.data_ptr(), ld, ml, j, wd.data_ptr(),
                      awd.data_ptr(), out.data_ptr(), ctypes.byref(segs), ws, wsb, table, rank,
                      world, cap, 6, err.data_ptr(), st)
        else:
            _lib.call("kls_gram_dcgs2", qb.data_ptr(), ld, ml, j, wd.data_ptr(), awd.data_ptr(),
                      out.data_ptr(), ctypes.byref(segs), ws, wsb, st)
        torch.cuda.synchronize()
        return out.cpu().numpy()

    segs = _lib.KlsSegs(m, 64, world, rank)
    lo, hi = runtime.seg_range(m, 64, world, rank)
    got = gram(lo, hi, segs, True)
    one = gram(0, m, _lib.KlsSegs(m, 64, 1, 0), False)
    left = np.hstack([Q, w[:, None]])
    want = np.concatenate([left.T @ w, left.T @ aw, [aw @ aw]])
    allg = [None] * world
    dist.all_gather_object(allg, got.tobytes())
    same = all(a == allg[0] for a in allg)
    close = np.allclose(got, want, rtol=1e-12, atol=1e-10)
    res.update(gram_close=bool(close), gram_bitwise_across_ranks=same,
               gram_bitwise_vs_one_rank=bool(np.array_equal(got, one)))
    ok = ok and close and same and np.array_equal(got, one) and int(err.item()) == 0

    dist.barrier()
    for r in range(world):
        if r != rank:
            _lib.call("kls_peer_buffer_close", ctypes.c_void_p(ptrs[r]))
    dist.barrier()
    _lib.call("kls_peer_buffer_free", mine)
    res["ok"] = bool(ok)
    if rank == 0:
        print(json.dumps(res), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
