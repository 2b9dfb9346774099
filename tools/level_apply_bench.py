"""Level-plan ILU0 application on C4: sync-free sweeps vs the wavefront kernels.

python tools/level_apply_bench.py [nx ny nz]
Each variant is checked bit for bit against the sync-free sweeps; prints
CUDA-event times and GB/s against SURVEY §8(d)'s algorithmic bytes.
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200 import ilu0 as I  # noqa: E402
from paper_2309_11488_b200.bridge import plan_device  # noqa: E402


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
a = P.generate(P.GeneratorSpec(*dims, block_size=int(os.environ.get("BS", "3")), seed=0)).a
n, nnz = a.num_block_rows, a.pattern.num_blocks
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
m = a.block_size * n
x = torch.rand(m, dtype=torch.float64, device="cuda")
alg = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 96 * n
out = {"dims": dims, "groups": plan.group_count}
ref = None
variants = [("syncfree", {"B2S_TILES": "0", "B2S_GW": "0"}),
            ("wavefront", {"B2S_TILES": "0", "B2S_GW": "1"})]
if os.environ.get("B2S_BENCH_TILES") == "1":
    variants += [("tiles_grid", {"B2S_TILES": "1", "B2S_GW": "0"})]
for name, env in variants:
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        f = I.factor_device(a, plan, bsr)
        z = torch.empty(m, dtype=torch.float64, device="cuda")
        t = ev_time(lambda: f.apply_device(x, z))
        zz = z.clone()
        if ref is None:
            ref = zz
        out[name] = {"us": round(t, 1), "gbs_alg": round(alg / t / 1e3, 1),
                     "bit_equal": bool(torch.equal(zz, ref)),
                     "tiles": getattr(f, "tile_shape", None) if f.tiles else None,
                     "gw": getattr(f, "gw_shape", None) if f.gw else None}
        del f
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
print(json.dumps(out))
