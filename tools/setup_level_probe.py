"""Level-plan setup on C4 (plan, factor, layouts, wavefront packing): CUDA
events per phase, previous solver freed first (as in bench.py).

python tools/setup_level_probe.py [level|color]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402

a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
backend = sys.argv[1] if len(sys.argv) > 1 else "level"
cfg = P.SolverConfig(backend=P.Backend.from_name(backend))
st = torch.cuda.current_stream()
out = {}
for gw in (("1", "0") if backend == "level" else ("1",)):
    os.environ["B2S_GW"] = gw
    ts = []
    solver = None
    for _ in range(6):
        solver = None
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        solver = DeviceSolver(a, bsr, cfg).setup()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[f"gw={gw}"] = {"setup_ms": sorted(ts)[len(ts) // 2], "all": [round(t, 2) for t in ts],
                       "gw": bool(solver.fact.gw)}
print(json.dumps(out))

# where the wavefront packing time goes
import time  # noqa: E402

from paper_2309_11488_b200 import ilu0 as I  # noqa: E402
os.environ["B2S_GW"] = "1"
orig = I._gw_plan
rec = []


def timed_gw(*args):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = orig(*args)
    torch.cuda.synchronize()
    rec.append((time.perf_counter() - t0) * 1e3)
    return out


I._gw_plan = timed_gw
for _ in range(4 if backend == "level" else 0):
    solver = None
    solver = DeviceSolver(a, bsr, cfg).setup()
print(json.dumps({"gw_plan_ms": [round(t, 3) for t in rec]}))
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    solver = None
    solver = DeviceSolver(a, bsr, cfg).setup()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
