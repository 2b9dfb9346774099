"""Pageable host -> device upload rate through the staging ring vs torch's
own copy (500 MB of fp64, like the C4 values).

B2S_STAGE_CHUNK_MB=.. B2S_STAGE_BUFS=.. B2S_STAGE_THREADS=.. python tools/stage_probe.py
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_11488_b200 import _device as D  # noqa: E402

a = np.random.default_rng(0).standard_normal(62_500_000)
src = torch.from_numpy(a)
dst = torch.empty(a.size, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
out = {"env": {k: os.environ.get(k) for k in ("B2S_STAGE_CHUNK_MB", "B2S_STAGE_BUFS",
                                               "B2S_STAGE_THREADS")}}
for name, fn in (("staged", lambda: D.staged_copy(dst, src, st)),
                 ("torch", lambda: dst.copy_(src))):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    out[name] = {"ms": round(min(ts) * 1e3, 2), "GBps": round(a.nbytes / min(ts) / 1e9, 1)}
print(json.dumps(out))
