"""Per-slice timeline of the wave tile kernel on C4 (level plan).

python tools/tile_trace.py [grid|range]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
mode = sys.argv[1] if len(sys.argv) > 1 else "grid"
os.environ["B2S_TILES"] = "1"
os.environ["B2S_TILES_GRID"] = "1" if mode == "grid" else "0"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import plan_device  # noqa: E402
from paper_2309_11488_b200.ilu0 import factor_device  # noqa: E402

a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
f = factor_device(a, plan, bsr)
assert f.tiles
T = f.tile_shape[0] * f.tile_shape[1] if len(f.tile_shape) == 2 else f.tile_shape[0]
buf = torch.zeros(2 * T * 1024 * 4, dtype=torch.int64, device="cuda")
D.lib().b2s_tiles_trace(f.tiles, buf.data_ptr(), 0)
m = a.num_block_rows * 3
x = torch.rand(m, dtype=torch.float64, device="cuda")
z = torch.empty(m, dtype=torch.float64, device="cuda")
for _ in range(3):
    f.apply_device(x, z)
torch.cuda.synchronize()
tr = buf.view(2, T, 1024, 4)[..., 2].cpu().numpy().astype(np.int64)
for d, name in ((0, "forward"), (1, "backward")):
    v = tr[d]
    t0 = v[v > 0].min()
    starts = np.array([(row[row > 0].min() - t0) if (row > 0).any() else -1 for row in v])
    ends = np.array([(row[row > 0].max() - t0) if (row > 0).any() else -1 for row in v])
    nsl = (v > 0).sum(axis=1)
    per = np.diff(v, axis=1)
    per = per[(per > 0) & (per < 1e7)]
    print(json.dumps({"sweep": name, "T": int(T), "slices_per_tile_max": int(nsl.max()),
                      "slices_per_tile_mean": float(nsl.mean()),
                      "tile_start_us": [float(np.percentile(starts, q)) / 1e3 for q in (0, 50, 100)],
                      "tile_end_us": [float(np.percentile(ends, q)) / 1e3 for q in (0, 50, 100)],
                      "slice_us_pct": [float(np.percentile(per, q)) / 1e3 for q in (10, 50, 90, 99)]}))
    # one tile's timeline (middle tile), first 40 slice gaps
    mid = T // 2
    row = v[mid][v[mid] > 0]
    print(json.dumps({"tile": int(mid), "gaps_us": [round(float(g) / 1e3, 2) for g in np.diff(row)[:60]]}))
