"""Randomised check of the wavefront kernels (sweeps + factorisation)
against the general paths, bit for bit: random grid shapes (incl. tile
remainders, thin and two-plane grids, wide grids on the shallow rings),
block sizes 1..4, level and sequential plans.

python tools/gw_stress.py [cases] [seed]
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for c in range(cases):
    shape = [int(v) for v in rng.integers(2, 48, size=3)]
    if rng.random() < 0.2:
        shape[rng.integers(0, 3)] = int(rng.integers(1, 3))
    if rng.random() < 0.15:
        shape = [int(rng.integers(180, 260)), int(rng.integers(60, 90)), int(rng.integers(1, 4))]
    bs = int(rng.integers(1, 5))
    kind = "level" if rng.random() < 0.7 else "sequential"
    a = P.generate(P.GeneratorSpec(*shape, block_size=bs, seed=c, diagonal_boost=1e-2)).a
    plan = P.level_schedule(a.pattern) if kind == "level" else P.sequential_plan(a.num_block_rows)
    r = P.BlockVector(rng.uniform(-1, 1, a.num_block_rows * bs), bs)
    out = {}
    for gw, fac in (("1", "1"), ("1", "0"), ("0", "0")):
        os.environ["B2S_GW"], os.environ["B2S_GW_FACTOR"] = gw, fac
        f = P.decompose(a, plan)
        lu = f.lu_device.vals[: f.lu_device.pat.nnz * bs * bs].cpu().numpy()
        out[(gw, fac)] = (lu, f.apply(r).data, f.gw is not None, f._gw_lazy is not None)
    ref = out[("0", "0")]
    ok = all(np.array_equal(v[0], ref[0]) and np.array_equal(v[1], ref[1]) for v in out.values())
    bad += not ok
    print(json.dumps({"case": c, "shape": shape, "b": bs, "plan": kind,
                      "gw": out[("1", "1")][2], "gw_factor": out[("1", "1")][3], "ok": ok}),
          flush=True)
print(json.dumps({"cases": cases, "failures": bad}))
