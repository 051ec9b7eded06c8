"""Multi-GPU parity through torchrun + NCCL (runs when >= 2 GPUs are
visible; the single-GPU round-end run skips it)."""

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


def test_peer_capi_without_symmetric_memory(cuda):
    """C-ABI peer buffers (kls_peer_buffer_alloc/open, IPC handles) carry the
    one-shot allreduce and the fused Gram + allreduce for a host that has no
    collective allocator (scripts/peer_capi_check.py)."""
    import torch

    n = min(torch.cuda.device_count(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29519",
           os.path.join(ROOT, "scripts", "peer_capi_check.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["world"] == n, res
