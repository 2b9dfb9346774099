"""Steady-state setup phase timings (each phase bracketed by a sync)."""
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


def phases(a, bsr, backend):
    import paper_2309_11488_b200.bridge as B
    import paper_2309_11488_b200.ilu0 as I
    import paper_2309_11488_b200.krylov as K
    t = {}

    def tick(name, fn, *args):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*args)
        torch.cuda.synchronize()
        t[name] = round((time.perf_counter() - t0) * 1e3, 3)
        return out
    plan = tick("plan", B.plan_device, backend, bsr.pat)
    f = tick("factor_device", I.factor_device, a, plan, bsr)
    tick("operator_layout", K.DeviceKrylov.build, a, f, f._a_perm)
    return t


def main():
    bundle = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
    a = bundle.a
    bsr = D.DevBSR.upload(a)
    for rep in range(3):
        for name, be in (("level", P.Backend.LEVEL_SCHEDULED), ("color", P.Backend.GRAPH_COLORED)):
            t = phases(a, bsr, be)
            if rep == 2:
                print(json.dumps({"backend": name, **t}), flush=True)
    # fine-grained: profile one level setup with torch profiler (kernel times)
    from torch.profiler import ProfilerActivity, profile
    for be in (P.Backend.GRAPH_COLORED, P.Backend.LEVEL_SCHEDULED):
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            DeviceSolver(a, bsr, P.SolverConfig(backend=be)).setup()
            torch.cuda.synchronize()
        print(be, prof.key_averages().table(sort_by="cuda_time_total", row_limit=14,
                                            max_name_column_width=40))


if __name__ == "__main__":
    main()
