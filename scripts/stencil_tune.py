"""Time the matrix-free stencil apply at config-3 size (m = 1.3e8); sweep the
x-chunk with KLS_STENCIL_XCHUNK and the variant with KLS_STENCIL=reg|smem.
"""
import os, sys, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_01253_b200 import laplace3d
dims = (496, 512, 512); m = dims[0]*dims[1]*dims[2]
op = laplace3d(*dims)
x = torch.randn(m, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): op.apply_into(x, y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): op.apply_into(x, y)
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e)/20*1e-3
print(json.dumps({"xchunk": os.environ.get("KLS_STENCIL_XCHUNK"), "ms": t*1e3, "GBs": 16*m/t/1e9}))
