"""Device-resident solve times of every BASELINE single-GPU configuration
(C1 4k, C2 NORNE-scale masked, C3 350k heterogeneous, C4 1M), level and
colour plans, tol 1e-8, plus SURVEY 8(d)'s variants: C1 and C4 at the
reference default tol 0.01, and C4 with diagonal boost 1e-2 (harder) at
tol 1e-8: setup, Krylov, iterations, Mcells/s.

python tools/configs_bench.py    (one JSON line per config and plan)
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200 import synthetic as S  # noqa: E402
from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402

CONFIGS = [   # (name, generator, tol)
    ("C1 20x20x10", lambda: P.generate(P.GeneratorSpec(20, 20, 10, seed=0)), 1e-8),
    ("C1 20x20x10", lambda: P.generate(P.GeneratorSpec(20, 20, 10, seed=0)), 1e-2),
    ("C2 46x112x22 masked", lambda: S.generate_masked(46, 112, 22, seed=2309), 1e-8),
    ("C3 92x224x17 heterogeneous", lambda: S.generate_heterogeneous(92, 224, 17, sigma_k=1.0,
                                                                    diagonal_boost=1e-2), 1e-8),
    ("C3s 92x224x17 heterogeneous sigma 2",
     lambda: S.generate_heterogeneous(92, 224, 17, sigma_k=2.0, diagonal_boost=1e-2), 1e-8, 400),
    ("C4 100x100x100", lambda: P.generate(P.GeneratorSpec(100, 100, 100, seed=0)), 1e-8),
    ("C4 100x100x100", lambda: P.generate(P.GeneratorSpec(100, 100, 100, seed=0)), 1e-2),
    ("C4 100x100x100 boost 1e-2",
     lambda: P.generate(P.GeneratorSpec(100, 100, 100, diagonal_boost=1e-2, seed=0)), 1e-8),
]
st = torch.cuda.current_stream()
for name, make, tol, *rest in CONFIGS:
    maxit = rest[0] if rest else 200
    bnd = make()
    a = bnd.a
    bsr = D.DevBSR.upload(a)
    rhs = D.f64(bnd.rhs.data, bsr.vals.device)
    for backend in ("level", "color"):
        cfg = P.SolverConfig(backend=P.Backend.from_name(backend),
                             stop=P.StoppingCriteria(tol, maxit))
        x = torch.zeros_like(rhs)
        times = []
        solver = None
        for rep in range(5):
            solver = None   # as bench.py: free the previous solver before the next setup
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            solver = DeviceSolver(a, bsr, cfg).setup()
            e1.record(st)
            x.zero_()
            res = solver.solve(rhs, x, cfg.stop, x0_zero=True)
            e2.record(st)
            torch.cuda.synchronize()
            if rep >= 2:   # two warm-up solves (module loading, allocator growth)
                times.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
        su = sum(t[0] for t in times) / len(times)
        kr = sum(t[1] for t in times) / len(times)
        solver_groups = solver.plan.group_count
        solver = None
        print(json.dumps({"config": name, "tol": tol, "maxit": maxit, "cells": a.num_block_rows,
                          "backend": backend,
                          "groups": solver_groups, "iterations": float(res.iterations),
                          "converged": bool(res.converged), "setup_ms": round(su, 3),
                          "krylov_ms": round(kr, 3), "solve_ms": round(su + kr, 3),
                          "mcells_per_s": round(a.num_block_rows / (su + kr) / 1e3, 2)}),
              flush=True)
