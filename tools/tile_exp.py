"""Tiled-sweep experiments: local pace (one tile) vs many tiles, warps per tile."""
import json
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


def run(dims, env):
    os.environ.update(env)
    bundle = P.generate(P.GeneratorSpec(*dims, seed=0))
    a = bundle.a
    bsr = D.DevBSR.upload(a)
    plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
    f = factor_device(a, plan, bsr)
    m = a.num_block_rows * 3
    x = torch.rand(m, dtype=torch.float64, device="cuda")
    z = torch.empty(m, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    best = 1e30
    for i in range(5):
        y = torch.empty(m, dtype=torch.float64, device="cuda")
        D.fill_sentinel(y, m)
        D.fill_sentinel(z, m)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        if f.tiles:
            D.check(D.lib().b2s_tiles_apply(3, f.tiles, D.ptr(x), D.ptr(y), D.ptr(z), 1,
                                            D.stream()), "apply")
        else:
            f.apply_device(x, z)
        e1.record(st)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    print(json.dumps({"dims": dims, "env": env, "tiled": bool(f.tiles),
                      "shape": getattr(f, "tile_shape", None), "levels": plan.group_count,
                      "apply_us": best, "us_per_level_per_sweep": best / 2 / plan.group_count}),
          flush=True)


if __name__ == "__main__":
    for w in ("8", "16", "32"):
        run((20, 20, 20), {"B2S_TILES": "1", "B2S_TILES_T": "1", "B2S_TILE_WARPS": w})
    run((20, 20, 20), {"B2S_TILES": "0"})
    for w in ("8", "16", "32"):
        run((40, 40, 40), {"B2S_TILES": "1", "B2S_TILES_T": "16", "B2S_TILE_WARPS": w})
    run((40, 40, 40), {"B2S_TILES": "0"})
    for w in ("16", "32"):
        run((100, 100, 100), {"B2S_TILES": "1", "B2S_TILES_T": "148", "B2S_TILE_WARPS": w})
