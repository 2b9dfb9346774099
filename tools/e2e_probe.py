"""Where the e2e time goes: solve_with_fallback's steps on pinned host
inputs, each bracketed by a host clock after a sync (C4, colour plan)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402

bundle = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = P.pin_host(bundle.a), P.pin_host(bundle.rhs)
cfg = P.SolverConfig(backend=P.Backend.GRAPH_COLORED, stop=P.StoppingCriteria(1e-8, 200))
dev = torch.device("cuda")
for rep in range(5):
    t = {}
    t0 = time.perf_counter()

    def tick(name):
        torch.cuda.synchronize()
        t[name] = round((time.perf_counter() - t0) * 1e3, 3)
    bsr = D.DevBSR.upload(a, overlap=True)
    tick("pattern_uploaded")
    rhs_d = D.f64(rhs.data, dev)
    x0 = torch.zeros(rhs.data.size, dtype=torch.float64, device=dev)
    s = DeviceSolver(a, bsr, cfg)
    from paper_2309_11488_b200.bridge import plan_device
    s.plan = plan_device(cfg.backend, bsr.pat)
    tick("analysis_done")
    bsr.wait_values()
    tick("values_landed")
    from paper_2309_11488_b200.ilu0 import factor_device
    from paper_2309_11488_b200.krylov import DeviceKrylov
    s.fact = factor_device(a, s.plan, bsr)
    tick("factored")
    s.krylov = DeviceKrylov.build(a, s.fact, s.fact._a_perm)
    tick("layout")
    res = s.solve(rhs_d, x0, cfg.stop)
    tick("krylov")
    x = D.to_host(x0, x0.numel())
    tick("d2h")
    if rep >= 2:
        print(json.dumps(t), flush=True)
    # the public call, for comparison
    t1 = time.perf_counter()
    P.solve_with_fallback(cfg, a, rhs)
    torch.cuda.synchronize()
    if rep >= 2:
        print(json.dumps({"solve_with_fallback_ms": (time.perf_counter() - t1) * 1e3}), flush=True)
