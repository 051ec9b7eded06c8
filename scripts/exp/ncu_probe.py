"""One launch each of K1 (gram_tma_kernel), K2 (dcgs2_update_tma_kernel) and
the stencil at config 3's m and j = 50, with the stencil's segment layout --
the target of the `ncu --set full` capture (profiles/ncu_summary_r02.json).

    ncu --set full -k regex:"gram_tma|dcgs2_update_tma|stencil7_smem" -c 3 \\
        python scripts/exp/ncu_probe.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2104_01253_b200 import _lib, laplace3d, runtime  # noqa: E402

j = int(os.environ.get("PROBE_J", "50"))
op = laplace3d(496, 512, 512)
m, ld = op.m_local, runtime.pad_rows(op.m_local)
Q = torch.randn((j + 1, ld), dtype=torch.float64, device="cuda")
w = torch.randn(ld, dtype=torch.float64, device="cuda")
aw = torch.randn(ld, dtype=torch.float64, device="cuda")
out = torch.empty(2 * j + 8, dtype=torch.float64, device="cuda")
coef = torch.randn(2 * j + 1, dtype=torch.float64, device="cuda") * 1e-3
ws, wsb = runtime.workspace(j + 1)
st = runtime.stream_handle()
_lib.call("kls_gram_dcgs2", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(), out.data_ptr(),
          op.segs.ptr, ws, wsb, st)
_lib.call("kls_dcgs2_update", Q.data_ptr(), ld, m, j, w.data_ptr(), aw.data_ptr(),
          coef.data_ptr(), 1.0, 1, op.segs.ptr, st)
y = torch.empty(m, dtype=torch.float64, device="cuda")
op.apply_into(w[:m], y)
torch.cuda.synchronize()
print("probe done", m, j)
