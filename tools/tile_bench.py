"""Tiled vs sync-free level-scheduled sweeps: time and bit-equality.

python tools/tile_bench.py [nx ny nz]
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import plan_device  # noqa: E402
from paper_2309_11488_b200.ilu0 import factor_device  # noqa: E402
from paper_2309_11488_b200.krylov import DeviceKrylov  # noqa: E402
from tools.sweep_bench import ev_time  # noqa: E402


def main():
    dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
    bundle = P.generate(P.GeneratorSpec(*dims, seed=0))
    a = bundle.a
    n, b, nnz = a.num_block_rows, a.block_size, a.pattern.num_blocks
    dev = torch.device("cuda", 0)
    bsr = D.DevBSR.upload(a)
    m = n * b
    x = torch.rand(m, dtype=torch.float64, device=dev)
    y = torch.empty(m, dtype=torch.float64, device=dev)
    apply_bytes = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 96 * n
    plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
    ref = None
    for cfg in ("0", "grid148", "grid120", "range148"):
        os.environ["B2S_TILES"] = "0" if cfg == "0" else "1"
        os.environ["B2S_TILES_GRID"] = "1" if cfg.startswith("grid") else "0"
        if cfg != "0":
            os.environ["B2S_TILES_T"] = cfg[-3:]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = factor_device(a, plan, bsr)
        torch.cuda.synchronize()
        tf = (time.perf_counter() - t0) * 1e3
        z = torch.empty(m, dtype=torch.float64, device=dev)
        f.apply_device(x, z)
        torch.cuda.synchronize()
        if ref is None:
            ref = z.clone()
        same = bool(torch.equal(z, ref))
        us = ev_time(lambda: f.apply_device(x, z)) - ev_time(
            lambda: (D.fill_sentinel(y, m), D.fill_sentinel(z, m)))
        kr = DeviceKrylov.build(a, f, f._a_perm)
        rhs = D.f64(bundle.rhs.data, dev)
        x0 = torch.zeros(m, dtype=torch.float64, device=dev)
        stop = P.StoppingCriteria(1e-8, 200)
        kr.solve(rhs, x0.clone(), stop)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = kr.solve(rhs, x0.clone(), stop)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        print(json.dumps({"tiles": cfg, "tiled": bool(f.tiles),
                          "shape": getattr(f, "tile_shape", None), "factor_ms": tf,
                          "ilu_apply_us": us, "gbs": apply_bytes / (us * 1e-6) / 1e9,
                          "bit_equal_to_sync_free": same, "krylov_ms": dt,
                          "its": res.iterations}), flush=True)


if __name__ == "__main__":
    main()
