"""HBM ceilings on this B200 for context: torch read-only reduction, copy,
and the K1/K2 kernels at j=100 (m=1.3e8)."""
import json, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) * 1e-3)
    return best
n = 1 << 31  # 16 GiB of fp64
x = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
r = {}
r["read_sum_GBs"] = 8 * n / t(lambda: x.sum()) / 1e9
r["copy_GBs"] = 16 * n / t(lambda: y.copy_(x)) / 1e9
r["fill_GBs"] = 8 * n / t(lambda: y.fill_(1.0)) / 1e9
print(json.dumps(r))
