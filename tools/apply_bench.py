"""Colour-plan ILU0 application: phased vs sync-free sweeps (C4 by default).

python tools/apply_bench.py [nx ny nz]
Checks the two paths agree bit for bit and prints CUDA-event times.
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


def ev_time(fn, reps=20, warm=3):
    st = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
a = P.generate(P.GeneratorSpec(*dims, seed=0)).a
n, nnz = a.num_block_rows, a.pattern.num_blocks
bsr = D.DevBSR.upload(a)
solver = DeviceSolver(a, bsr, P.SolverConfig(backend=P.Backend.GRAPH_COLORED)).setup()
f = solver.fact
m = 3 * n
x = torch.rand(m, dtype=torch.float64, device="cuda")
z1 = torch.empty(m, dtype=torch.float64, device="cuda")
z0 = torch.empty(m, dtype=torch.float64, device="cuda")
assert f.phased, "colour plan should take the phased sweeps"
t_ph = ev_time(lambda: f.apply_device(x, z1))
f.phased = False
t_sf = ev_time(lambda: f.apply_device(x, z0))
f.phased = True
same = bool(torch.equal(z0, z1))
alg = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 96 * n
lean = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 48 * n   # r in, z out only
print(json.dumps({"dims": dims, "bit_equal": same, "phased_us": t_ph, "syncfree_us": t_sf,
                  "phased_gbs_alg": alg / t_ph / 1e3, "phased_gbs_lean": lean / t_ph / 1e3,
                  "syncfree_gbs_alg": alg / t_sf / 1e3}))
