"""Sharded solve on one GPU: where does a step go?  (setup, rhs upload, the
peer-memory device loop vs the host-driven loop)

python tools/mesh_probe.py [world] [backend]
"""
import json
import os
import sys
import time
from pathlib import Path

# one hardware queue per shard stream (solve_shards_mesh checks it)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200.distributed import (local_solver, solve_shards,  # noqa: E402
                                               solve_shards_mesh)

world = int(sys.argv[1]) if len(sys.argv) > 1 else 1
backend = P.Backend.from_name(sys.argv[2] if len(sys.argv) > 2 else "color")
spec = P.GeneratorSpec(100, 100, 100 * world, seed=0)
stop = P.StoppingCriteria(1e-8, 200)
shards, comm = local_solver(spec, world, backend)


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return round(best * 1e3, 3), out


res = {"world": world, "backend": backend.value}
res["setup_ms"], _ = t(lambda: [s.setup(backend) for s in shards])
res["mesh_solve_ms"], (rep, _) = t(lambda: solve_shards_mesh(shards, stop))
res["mesh_its"] = rep.iterations
res["host_loop_ms"], (rep2, _) = t(lambda: solve_shards(shards, comm, stop))
res["host_its"] = rep2.iterations
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    solve_shards_mesh(shards, stop)
    torch.cuda.synchronize()
print(json.dumps(res), flush=True)
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=16, max_name_column_width=50))
