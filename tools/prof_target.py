"""Small driver for ncu captures: a few SpMV + ILU0 applications on C4.

python tools/prof_target.py [color|level]
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
bundle = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
a = bundle.a
bsr = D.DevBSR.upload(a)
solver = DeviceSolver(a, bsr, P.SolverConfig(backend=P.Backend.from_name(backend))).setup()
f, kr = solver.fact, solver.krylov
m = a.num_block_rows * 3
x = torch.rand(m, dtype=torch.float64, device="cuda")
y = torch.empty(m, dtype=torch.float64, device="cuda")
z = torch.empty(m, dtype=torch.float64, device="cuda")
parts = torch.empty(D.NPARTS, dtype=torch.float64, device="cuda")
for _ in range(4):
    D.spmv(kr.smap, kr.a, 3, x, y, 1, x, parts)
    f.apply_device(x, z)
torch.cuda.synchronize()
print("done", backend)
