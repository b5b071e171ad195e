"""Pinned device->host copy bandwidth of one GPU (the e2e path's bound):
1.59 GB (c3's images per step) in one copy and in 8 / 32 chunks."""
import json
import torch

n = 132710400 * 3
src = torch.empty(n, dtype=torch.int32, device="cuda")
dst = torch.empty(n, dtype=torch.int32, pin_memory=True)
res = {}
for chunks in (1, 8, 32):
    step = (n + chunks - 1) // chunks
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(0, n, step):
            dst[i:i + step].copy_(src[i:i + step], non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = max(best, 4 * n / (a.elapsed_time(b) / 1e3) / 1e9)
    res[f"d2h_gbs_{chunks}"] = round(best, 2)
print(json.dumps(res))
