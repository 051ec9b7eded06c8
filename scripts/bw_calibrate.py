import torch, json
for mb in (24, 56, 216, 416, 1000, 4000):
    n = mb * 1024 * 1024 // 8
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    for _ in range(3): x.sum()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 30
    e0.record()
    for _ in range(reps): x.sum()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(json.dumps({"MB": mb, "sum_us": round(us, 2), "TBs": round(n * 8 / us / 1e6, 2), "ideal_us_7.3": round(n*8/7.3e6, 2)}))
