"""e2e phase breakdown of solve_with_fallback (pinned C4, colour) with
B2S_TRACE=1: host and GPU time per phase."""
import json
import os
import sys
import time
from pathlib import Path

os.environ["B2S_TRACE"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402

b = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = P.pin_host(b.a), P.pin_host(b.rhs)
cfg = P.SolverConfig(backend=P.Backend.GRAPH_COLORED, stop=P.StoppingCriteria(1e-8, 200))
x = None
for rep in range(5):
    x = None   # as bench.py: the previous solution is released first (its pinned block is reused)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, r = P.solve_with_fallback(cfg, a, rhs)
    wall = (time.perf_counter() - t0) * 1e3
    if rep:
        print(json.dumps({"wall_ms": round(wall, 3), **r.phases}), flush=True)
