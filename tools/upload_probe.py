"""Timeline of the e2e upload (pinned C4 system): pattern (int64) copy +
device narrowing, values copy on the side stream, rhs."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402

b = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = P.pin_host(b.a), P.pin_host(b.rhs)
for rep in range(4):
    torch.cuda.synchronize()
    t = {}
    t0 = time.perf_counter()
    pat = D.DevPattern.upload(a.pattern)
    t["pattern_host_returns"] = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    t["pattern_done"] = (time.perf_counter() - t0) * 1e3
    t1 = time.perf_counter()
    v = torch.empty(a.values.size, dtype=torch.float64, device="cuda")
    v.copy_(torch.from_numpy(a.values), non_blocking=True)
    torch.cuda.synchronize()
    t["values_ms"] = (time.perf_counter() - t1) * 1e3
    t2 = time.perf_counter()
    bsr = D.DevBSR.upload(a, overlap=True)
    t["upload_host_returns"] = (time.perf_counter() - t2) * 1e3
    bsr.wait_values()
    torch.cuda.synchronize()
    t["upload_total"] = (time.perf_counter() - t2) * 1e3
    if rep:
        print(json.dumps({k: round(x, 3) for k, x in t.items()}), flush=True)
