"""C4 solve with SolverConfig(jacobi_partitions=k):
host weights + greedy partition (vectorised numpy + the C++ walk), the
relaxed matrix dropped from the resident operator on the device, then the
usual device pipeline.  Prints one JSON line per backend.

python tools/jacobi_bench.py [k] [reps]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import jacobi as J  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 150
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = P.pin_host(g.a), P.pin_host(g.rhs)
t0 = time.perf_counter()
ew = J._edge_weights(a)
t1 = time.perf_counter()
part = J.partition(a.pattern, ew, k)
t2 = time.perf_counter()
for backend in ("color", "level"):
    cfg = P.SolverConfig(backend=P.Backend.from_name(backend), jacobi_partitions=k,
                         stop=P.StoppingCriteria(1e-8, 200))
    P.solve_with_fallback(cfg, a, rhs)
    torch.cuda.synchronize()
    ts, reps_out = [], None
    for _ in range(reps):
        s0 = time.perf_counter()
        x, rep = P.solve_with_fallback(cfg, a, rhs)
        ts.append(time.perf_counter() - s0)
        reps_out = rep
    plain = P.solve_with_fallback(P.SolverConfig(backend=P.Backend.from_name(backend),
                                                 stop=P.StoppingCriteria(1e-8, 200)), a, rhs)[1]
    print(json.dumps({"backend": backend, "k": k, "cells": a.num_block_rows,
                      "host_weights_s": t1 - t0, "host_partition_s": t2 - t1,
                      "call_s": min(ts), "iterations": reps_out.iterations,
                      "groups": reps_out.group_count, "converged": reps_out.converged,
                      "setup_s": reps_out.setup_elapsed, "krylov_s": reps_out.elapsed,
                      "unrelaxed_iterations": plain.iterations,
                      "unrelaxed_groups": plain.group_count}), flush=True)
