"""Per-iteration cost of the device BiCGStab loop on C4 (setup excluded).

python tools/krylov_bench.py [color|level] [iters] [nx,ny,nz]
Runs a fixed number of iterations (tol 1e-30 so the budget ends the solve)
and prints ms per iteration (CUDA events on the solve stream).
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402

backend = sys.argv[1] if len(sys.argv) > 1 else "color"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 60
dims = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else (100, 100, 100)
bundle = P.generate(P.GeneratorSpec(*dims, seed=0))
a, rhs = bundle.a, bundle.rhs
bsr = D.DevBSR.upload(a)
solver = DeviceSolver(a, bsr, P.SolverConfig(backend=P.Backend.from_name(backend))).setup()
kr = solver.krylov
n = a.num_block_rows
iperm = solver.plan.device("inverse_permutation")
bp = D.gather_rows(D.f64(rhs.data, "cuda"), iperm, n, 3)
stop = P.StoppingCriteria(1e-30, iters)
st = torch.cuda.current_stream()
out = []
for rep in range(4):
    x = torch.zeros(3 * n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    res = kr.solve(bp, x, stop)
    e1.record(st)
    torch.cuda.synchronize()
    out.append(e0.elapsed_time(e1))
print(json.dumps({"backend": backend, "dims": dims, "iterations": res.iterations, "reason": res.reason,
                  "ms": out, "us_per_iter": min(out) / max(res.iterations, 1) * 1e3,
                  "kernels_per_iteration": res.kernels_per_iteration,
                  "graph_launches": res.graph_launches}))
