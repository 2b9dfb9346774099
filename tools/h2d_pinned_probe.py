"""Pinned host -> device copy rate: one copy vs several concurrent chunks."""
import json
import time

import torch

n = 62_460_000   # C4 values (6.94M blocks x 9 doubles, 500 MB)
src = torch.empty(n, dtype=torch.float64, pin_memory=True)
src.uniform_()
dst = torch.empty(n, dtype=torch.float64, device="cuda")
out = {}
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunks = [(i * n // k, (i + 1) * n // k) for i in range(k)]
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s, (a, b) in zip(streams, chunks):
            with torch.cuda.stream(s):
                dst[a:b].copy_(src[a:b], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    out[f"streams_{k}"] = {"ms": round(best * 1e3, 2), "GBs": round(n * 8 / best / 1e9, 1)}
d2h = torch.empty(3_000_000, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d2h.copy_(dst[:3_000_000], non_blocking=True)
torch.cuda.synchronize()
out["d2h_24MB_ms"] = round((time.perf_counter() - t0) / 10 * 1e3, 3)
print(json.dumps(out))
