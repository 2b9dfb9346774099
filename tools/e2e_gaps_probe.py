"""Device-idle gaps inside one end-to-end C4 solve (solve_with_fallback from
page-locked host arrays): every gap > 20 us between consecutive GPU
activities (kernels and copies, all streams) with the activity after it.

python tools/e2e_gaps_probe.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402

g = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = P.pin_host(g.a), P.pin_host(g.rhs)
cfg = P.SolverConfig(backend=P.Backend.GRAPH_COLORED, stop=P.StoppingCriteria(1e-8, 200))
for _ in range(3):
    P.solve_with_fallback(cfg, a, rhs)
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    P.solve_with_fallback(cfg, a, rhs)
    torch.cuda.synchronize()
dev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
t0, last = dev[0].time_range.start, dev[0].time_range.end
idle = 0.0
for e in dev[1:]:
    gap = e.time_range.start - last
    if gap > 20:
        idle += gap
        print(json.dumps({"gap_us": round(gap, 1), "at_us": round(e.time_range.start - t0, 1),
                          "next": e.name[:70]}))
    last = max(last, e.time_range.end)
print(json.dumps({"span_us": round(last - t0, 1), "idle_over_20us": round(idle, 1)}))
