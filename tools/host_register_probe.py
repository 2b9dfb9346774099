"""Pageable numpy -> device: cudaHostRegister (pin in place) + plain DMA +
unregister, against the staging ring, for 500 MB (the C4 values).

python tools/host_register_probe.py
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_11488_b200 import _device as D  # noqa: E402

n = 62_500_000
rt = torch.cuda.cudart()
out = {}
dst = torch.empty(n, dtype=torch.float64, device="cuda")
for rep in range(3):
    a = np.random.default_rng(rep).standard_normal(n)     # fresh pageable array
    src = torch.from_numpy(a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(src.data_ptr(), src.numel() * 8, 0)
    t1 = time.perf_counter()
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    rt.cudaHostUnregister(src.data_ptr())
    t3 = time.perf_counter()
    ok = bool(torch.equal(dst.cpu(), src))
    b = np.random.default_rng(10 + rep).standard_normal(n)
    srcb = torch.from_numpy(b)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    D.staged_copy(dst, srcb, torch.cuda.current_stream())
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    out[f"rep{rep}"] = {"register_ms": round((t1 - t0) * 1e3, 2), "dma_ms": round((t2 - t1) * 1e3, 2),
                        "unregister_ms": round((t3 - t2) * 1e3, 2), "rc": int(rc), "exact": ok,
                        "staged_ms": round((t5 - t4) * 1e3, 2)}
print(json.dumps(out))
