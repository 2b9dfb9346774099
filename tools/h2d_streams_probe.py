"""Page-locked host -> device copy rate of 500 MB with the copy split over
1, 2 or 4 streams (DMA engines working in parallel on one PCIe link?).

python tools/h2d_streams_probe.py
"""
import json
import time

import torch

n = 62_500_000
src = torch.empty(n, dtype=torch.float64, pin_memory=True)
src.uniform_()
dst = torch.empty(n, dtype=torch.float64, device="cuda")
out = {}
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]

    def go():
        for st, (lo, hi) in zip(streams, parts):
            with torch.cuda.stream(st):
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
        torch.cuda.synchronize()
    go()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        go()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    out[f"streams={k}"] = {"ms": round(t * 1e3, 3), "GBps": round(n * 8 / t / 1e9, 1)}
# D2H too
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h.copy_(dst)
torch.cuda.synchronize()
t0 = time.perf_counter()
h.copy_(dst, non_blocking=True)
torch.cuda.synchronize()
out["d2h"] = {"GBps": round(n * 8 / (time.perf_counter() - t0) / 1e9, 1)}
print(json.dumps(out))
