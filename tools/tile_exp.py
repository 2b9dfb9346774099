"""Tiled step kernels on C4: where does a step's time go?

python tools/tile_exp.py
  cold : normal application (outputs sentinel-filled, cross-tile inputs polled)
  warm : outputs already hold the result, so every cross-tile poll succeeds on
         its first load -- the step time without waiting on other tiles
  nopoll (dbg 1): cross-tile inputs skipped; pipe (dbg 2): no row work at all
Prints per-step gap percentiles (globaltimer, consumer thread 0) and times.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import plan_device  # noqa: E402
from paper_2309_11488_b200.ilu0 import factor_device  # noqa: E402

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
a = P.generate(P.GeneratorSpec(*dims, seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
f = factor_device(a, plan, bsr)
assert f.tiles
T = f.tile_shape[0] * f.tile_shape[1] if len(f.tile_shape) == 2 else f.tile_shape[0]
m = a.num_block_rows * 3
x = torch.rand(m, dtype=torch.float64, device="cuda")
y = torch.empty(m, dtype=torch.float64, device="cuda")
z = torch.empty(m, dtype=torch.float64, device="cuda")
buf = torch.zeros(2 * T * 1024 * 4, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()


def run(warm):
    if not warm:
        D.fill_sentinel(y, m)
        D.fill_sentinel(z, m)
    D.check(D.lib().b2s_tiles_apply(3, f.tiles, D.ptr(x), D.ptr(y), D.ptr(z), 0, D.stream()),
            "tiles_apply")


def timed(warm, reps=10):
    run(warm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        run(warm)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


out = {"T": T}
for mode, warm, dbg in (("cold", False, 0), ("cold_nopf", False, 4), ("warm", True, 0),
                        ("nopoll", False, 1), ("pipe", False, 2)):
    D.lib().b2s_tiles_trace(f.tiles, None, dbg)
    out[mode + "_us"] = round(timed(warm), 1)
    buf.zero_()
    D.lib().b2s_tiles_trace(f.tiles, buf.data_ptr(), dbg)
    run(warm)
    torch.cuda.synchronize()
    tr = buf.view(2, T, 1024, 4).cpu().numpy().astype(np.int64)
    for d, name in ((0, "fwd"), (1, "bwd")):
        v = tr[d]
        ok = (v > 0).all(axis=2)
        out[f"{mode}_{name}_nonzero"] = [int((v[..., k] > 0).sum()) for k in range(4)]
        if not ok.any():
            continue
        t0 = v[..., 0][ok].min()
        ready = v[..., 1] - v[..., 0]
        bar = v[..., 2] - v[..., 1]
        work = v[..., 3] - v[..., 2]
        gap = np.diff(v[..., 2], axis=1)
        okg = ok[:, 1:] & ok[:, :-1]

        def pct(a, m):
            a = a[m]
            return [round(float(np.percentile(a, q)) / 1e3, 3) for q in (10, 50, 90)]
        if mode in ("cold", "pipe"):
            for tt in (0, 1, T // 2, T - 1):
                g = np.diff(v[tt, :, 2])[:30] / 1e3
                wk = (v[tt, :30, 3] - v[tt, :30, 2]) / 1e3
                rd = (v[tt, :30, 1] - v[tt, :30, 0]) / 1e3
                out[f"{mode}_{name}_tile{tt}"] = {"gap": [round(float(x), 2) for x in g],
                                                  "work": [round(float(x), 2) for x in wk],
                                                  "issue_to_ready": [round(float(x), 2) for x in rd]}
        out[f"{mode}_{name}"] = {"issue_to_ready": pct(ready, ok), "ready_to_bar": pct(bar, ok),
                                 "work": pct(work, ok), "step_gap": pct(gap, okg),
                                 "end_us": round(float((v[..., 3][ok].max() - t0)) / 1e3, 1)}
    D.lib().b2s_tiles_trace(f.tiles, None, 0)
print(json.dumps(out, indent=1))
