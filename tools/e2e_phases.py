"""Phase times of the end-to-end C4 solve through solve_with_fallback
(host arrays in, host x out), page-locked or pageable inputs.

python tools/e2e_phases.py [pinned|pageable] [steps] [color|level]
Prints one JSON line per step: wall ms and {phase: (host_ms, gpu_ms)}
(paper_2309_11488_b200/trace.py; B2S_TRACE is switched on here).
"""
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

mode = sys.argv[1] if len(sys.argv) > 1 else "pinned"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
g = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = g.a, g.rhs
if mode == "pinned":
    a, rhs = P.pin_host(a), P.pin_host(rhs)
backend = sys.argv[3] if len(sys.argv) > 3 else "color"
cfg = P.SolverConfig(backend=P.Backend.from_name(backend), stop=P.StoppingCriteria(1e-8, 200))
if os.environ.get("E2E_MEMHIST"):
    torch.cuda.memory._record_memory_history(max_entries=200000)
for i in range(steps + 2):
    torch.cuda.synchronize()
    m0 = torch.cuda.memory_stats()
    t0 = time.perf_counter()
    x, rep = P.solve_with_fallback(cfg, a, rhs)
    ms = (time.perf_counter() - t0) * 1e3
    m1 = torch.cuda.memory_stats()
    alloc = {k: m1.get(k, 0) - m0.get(k, 0) for k in ("num_device_alloc", "num_device_free",
                                                      "num_alloc_retries")}
    alloc["reserved_gb"] = round(m1.get("reserved_bytes.all.current", 0) / 2**30, 3)
    alloc["allocated_gb"] = round(m1.get("allocated_bytes.all.current", 0) / 2**30, 3)
    if i >= 2:
        ph = {k: [round(v[0], 3), round(v[1], 3)] for k, v in (rep.phases or {}).items()}
        print(json.dumps({"mode": mode, "backend": backend, "wall_ms": round(ms, 3), "iterations": rep.iterations,
                          "phases": ph, "allocator": alloc}))
if os.environ.get("E2E_MEMHIST"):
    # the live blocks after the last step, largest first, with their stacks
    snap = torch.cuda.memory._snapshot()
    blocks = []
    for seg in snap["segments"]:
        for b in seg["blocks"]:
            if b["state"] == "active_allocated":
                fr = [f"{f['filename'].split('/')[-1]}:{f['line']}:{f['name']}" for f in b.get("frames", [])
                      if "paper_2309" in f["filename"] or "tools" in f["filename"]]
                blocks.append((b["size"], fr[:6]))
    blocks.sort(key=lambda t: -t[0])
    for size, fr in blocks[:25]:
        print(json.dumps({"mb": round(size / 2**20, 2), "stack": fr}))
