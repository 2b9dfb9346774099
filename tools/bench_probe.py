"""Reproduce bench.py's step loop and split the setup into phases
(CUDA events + host clock per phase, no extra syncs inside a step)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
import paper_2309_11488_b200.bridge as B  # noqa: E402
import paper_2309_11488_b200.ilu0 as I  # noqa: E402
import paper_2309_11488_b200.krylov as K  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402

backend = sys.argv[1] if len(sys.argv) > 1 else "color"
keep = "--keep" in sys.argv
bundle = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a, rhs = bundle.a, bundle.rhs
bsr = D.DevBSR.upload(a)
st = torch.cuda.current_stream()
be = P.Backend.from_name(backend)
prev = None
for it in range(8):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    h = [time.perf_counter()]
    ev[0].record(st)
    plan = B.plan_device(be, bsr.pat)
    ev[1].record(st); h.append(time.perf_counter())
    f = I.factor_device(a, plan, bsr)
    ev[2].record(st); h.append(time.perf_counter())
    kr = K.DeviceKrylov.build(a, f, f._a_perm)
    ev[3].record(st); h.append(time.perf_counter())
    torch.cuda.synchronize()
    h.append(time.perf_counter())
    out = {"it": it, "gpu_ms": [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(3)],
           "host_ms": [round((h[i + 1] - h[i]) * 1e3, 3) for i in range(4)],
           "mem_gb": round(torch.cuda.memory_allocated() / 1e9, 2),
           "reserved_gb": round(torch.cuda.memory_reserved() / 1e9, 2)}
    print(json.dumps(out), flush=True)
    if keep:
        prev = (plan, f, kr)
