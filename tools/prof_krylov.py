"""One C4 colour solve (device-resident) -- a driver for ncu captures of the
Krylov iteration's kernels, e.g.
  ncu --set full -k regex:k_spmv --launch-skip 6 --launch-count 2 python tools/prof_krylov.py
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402

backend = sys.argv[1] if len(sys.argv) > 1 else "color"
g = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
bsr = D.DevBSR.upload(g.a)
cfg = P.SolverConfig(backend=P.Backend.from_name(backend), stop=P.StoppingCriteria(1e-8, 200))
solver = DeviceSolver(g.a, bsr, cfg).setup()
rhs = D.f64(g.rhs.data, bsr.vals.device)
x = torch.zeros_like(rhs)
res = solver.solve(rhs, x, cfg.stop)
torch.cuda.synchronize()
print("iterations", res.iterations)
