"""Multi-rank parity through torchrun.  The NCCL tests need >= 2 GPUs; the
rank-invariance and C-ABI peer tests also run with several ranks SHARING
one GPU (gloo bootstrap + CUDA-IPC peer buffers), so the single-GPU
round-end run exercises the sharded path too."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("want", [4, 3])
def test_row_sharded_parity_nccl(cuda, want):
    """4 ranks (or all there are), and 3 ranks: uneven row blocks."""
    import torch

    have = torch.cuda.device_count()
    n = min(have, want)
    if n < 2 or (want == 3 and have < 3):
        pytest.skip("needs >= 2 GPUs (3 for the uneven split)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={29517 + want}",
           os.path.join(ROOT, "scripts", "dist_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["world"] == n, res


def _torchrun(n, port, script, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "scripts", script),
           *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_rank_count_invariance(cuda, tmp_path):
    """The same problems on 1, 2 and 3 ranks (on however many GPUs there are:
    ranks share a GPU when there are fewer) give BITWISE identical results:
    Arnoldi H and basis rows (stencil, host and device CSR, DCGS2 / CGS2),
    GMRES iterations and histories, Krylov-Schur lock history and values,
    QR's R (scripts/rank_invariance.py)."""
    outs = []
    for n in (1, 2, 3):
        out = str(tmp_path / f"rankinv_{n}.npz")
        r = _torchrun(n, 29530 + n, "rank_invariance.py", "--out", out, timeout=900)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        outs.append(out)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "rank_invariance.py"),
                        "--compare", *outs], capture_output=True, text=True, timeout=300, cwd=ROOT)
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert r.returncode == 0 and res["ok"], res


def test_peer_capi_without_symmetric_memory(cuda):
    """C-ABI peer buffers (kls_peer_buffer_alloc/open, IPC handles) carry the
    segment-tree combine and the fused Gram + combine for a host that has no
    collective allocator, bitwise equal to one rank (scripts/peer_capi_check.py);
    two ranks per GPU when there is one GPU."""
    import torch

    n = max(2, min(torch.cuda.device_count(), 4))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29519",
           os.path.join(ROOT, "scripts", "peer_capi_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["world"] == n, res
