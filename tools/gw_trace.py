"""Per-step timeline of the wavefront sweeps (csrc/gridwave.cu) on C4:
start offsets of the tiles and the step time inside one tile.

B2S_GW_TRACE=1 python tools/gw_trace.py [nx ny nz [krylov]]
"""
import ctypes as C
import json
import os
import sys
from pathlib import Path

os.environ["B2S_GW_TRACE"] = "1"
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200 import ilu0 as I  # noqa: E402
from paper_2309_11488_b200.bridge import plan_device  # noqa: E402

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
a = P.generate(P.GeneratorSpec(*dims, block_size=int(os.environ.get("BS", "3")), seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
f = I.factor_device(a, plan, bsr)
assert f.gw, "wavefront sweeps not engaged"
if len(sys.argv) > 4 and sys.argv[4] == "krylov":
    # the last sweeps of a device BiCGStab solve (one CUDA graph per iteration)
    from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402
    g = P.generate(P.GeneratorSpec(*dims, seed=0))
    solver = DeviceSolver(g.a, bsr, P.SolverConfig(backend=P.Backend.LEVEL_SCHEDULED)).setup()
    f = solver.fact
    x = torch.zeros(3 * a.num_block_rows, dtype=torch.float64, device="cuda")
    for _ in range(int(os.environ.get("GW_TRACE_SOLVES", "1"))):
        x.zero_()
        solver.solve(D.f64(g.rhs.data, "cuda"), x, P.StoppingCriteria(1e-30, 12))
else:
    x = torch.rand(a.block_size * a.num_block_rows, dtype=torch.float64, device="cuda")
    z = torch.empty_like(x)
    for _ in range(3):
        f.apply_device(x, z)
torch.cuda.synchronize()
cnt = C.c_longlong(0)
shape = (C.c_int * 5)()
D.lib().b2s_gw_trace(C.c_void_p(f.gw), None, 0, C.byref(cnt), shape)
TX, TY, S, wx, wy = list(shape)
KTL = 64
buf = np.zeros(cnt.value + TX * TY * (1 + 4 * KTL), dtype=np.uint64)
rc = D.lib().b2s_gw_trace(C.c_void_p(f.gw), buf.ctypes.data, buf.size, C.byref(cnt), shape)
tl = buf[cnt.value:]
buf = buf[:cnt.value]
tr = buf.astype(np.int64).reshape(2, TY, TX, S)
out = {"dims": dims, "tiles": [TX, TY], "S": S}
for d, name in ((0, "fwd"), (1, "bwd")):
    t = tr[d]
    valid = t > 0
    t0 = t[valid].min()
    first = np.where(valid, t, np.iinfo(np.int64).max).min(axis=2) - t0   # per tile first step end
    last = t.max(axis=2) - t0
    steps = np.diff(t[0, 0][t[0, 0] > 0])
    mid = np.diff(t[TY // 2, TX // 2][t[TY // 2, TX // 2] > 0])
    out[name] = {"span_us": float((t[valid].max() - t0) / 1e3),
                 "first_step_end_us": {"t00": float(first[0, 0] / 1e3),
                                       "last_tile": float(first[-1, -1] / 1e3) if d == 0 else
                                       float(first[0, 0] / 1e3),
                                       "row0_by_tx": (first[0, :] / 1e3).round(1).tolist(),
                                       "col0_by_ty": (first[:, 0] / 1e3).round(1).tolist()},
                 "tile00_step_us_median": float(np.median(steps) / 1e3) if steps.size else None,
                 "tilemid_step_us_median": float(np.median(mid) / 1e3) if mid.size else None,
                 "tilemid_step_us_p90": float(np.percentile(mid, 90) / 1e3) if mid.size else None}
# per-launch timeline (trace builds): spans of the last sweep launches
nl = int(tl[:TX * TY].min())
if nl > 0:
    rec = tl[TX * TY:].astype(np.int64).reshape(TX * TY, KTL, 4)
    k = min(nl, KTL)
    idx = [(nl - k + i) % KTL for i in range(k)]
    r = rec[:, idx]                                # [T][k][4]
    t0 = r[:, 0, 0].min()
    launches = []
    for i in range(k):
        e, w, x = r[:, i, 0], r[:, i, 1], r[:, i, 2]
        launches.append({"dir": int(r[0, i, 3]),
                         "entry_first_us": round((e.min() - t0) / 1e3, 1),
                         "entry_last_us": round((e.max() - t0) / 1e3, 1),
                         "wait_last_us": round((w.max() - t0) / 1e3, 1),
                         "exit_last_us": round((x.max() - t0) / 1e3, 1) if x.max() > 0 else None})
    out["launches"] = launches
print(json.dumps(out))
