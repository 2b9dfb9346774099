"""Time the tiled sweep kernels alone (one config) -- for ncu captures."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import plan_device  # noqa: E402
from paper_2309_11488_b200.ilu0 import factor_device  # noqa: E402

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
bundle = P.generate(P.GeneratorSpec(*dims, seed=0))
a = bundle.a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
f = factor_device(a, plan, bsr)
print("tiles", bool(f.tiles), getattr(f, "tile_shape", None), flush=True)
m = a.num_block_rows * 3
x = torch.rand(m, dtype=torch.float64, device="cuda")
z = torch.empty(m, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    y = torch.empty(m, dtype=torch.float64, device="cuda")
    D.fill_sentinel(y, m)
    D.fill_sentinel(z, m)
    e0.record(st)
    D.check(D.lib().b2s_tiles_apply(3, f.tiles, D.ptr(x), D.ptr(y), D.ptr(z), 1, D.stream())
            if f.tiles else 0, "apply")
    e1.record(st)
    torch.cuda.synchronize()
    print("apply_us", e0.elapsed_time(e1) * 1e3, flush=True)
