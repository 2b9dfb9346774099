"""Micro-benchmark of the hot kernels and the setup phases on one system.

python tools/sweep_bench.py [nx ny nz]   (default 100 100 100)
Prints one JSON line per measurement (CUDA-event timed on the current stream).
"""

import json
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


def ev_time(fn, reps=10, warm=2):
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
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (100, 100, 100)
    bundle = P.generate(P.GeneratorSpec(*dims, seed=0))
    a = bundle.a
    n, b, nnz = a.num_block_rows, a.block_size, a.pattern.num_blocks
    dev = torch.device("cuda", 0)
    t = time.perf_counter()
    bsr = D.DevBSR.upload(a)
    torch.cuda.synchronize()
    print(json.dumps({"upload_ms": (time.perf_counter() - t) * 1e3}))
    m = n * b
    x = torch.rand(m, dtype=torch.float64, device=dev)
    z = torch.empty(m, dtype=torch.float64, device=dev)
    y = torch.empty(m, dtype=torch.float64, device=dev)
    spmv_bytes = nnz * 76 + (n + 1) * 4 + 48 * n
    apply_bytes = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 96 * n
    for name, backend in (("level", P.Backend.LEVEL_SCHEDULED), ("color", P.Backend.GRAPH_COLORED)):
        phases = {}
        t = time.perf_counter()
        plan = plan_device(backend, bsr.pat)
        torch.cuda.synchronize()
        phases["plan_ms"] = (time.perf_counter() - t) * 1e3
        t = time.perf_counter()
        f = factor_device(a, plan, bsr)
        torch.cuda.synchronize()
        phases["factor_total_ms"] = (time.perf_counter() - t) * 1e3
        t = time.perf_counter()
        kr = DeviceKrylov.build(a, f, f._a_perm)
        torch.cuda.synchronize()
        phases["operator_layout_ms"] = (time.perf_counter() - t) * 1e3
        print(json.dumps({"plan": name, "groups": plan.group_count, **phases}))
        for flags in (0, 4, 0x14, 0x24, 0x414, 0x10):
            f.sweep_flags = flags
            us_apply = ev_time(lambda: f.apply_device(x, z))
            us_fill = ev_time(lambda: (D.fill_sentinel(y, m), D.fill_sentinel(z, m)))
            us = us_apply - us_fill
            print(json.dumps({"plan": name, "flags": flags, "ilu_apply_us": us,
                              "gbs": apply_bytes / (us * 1e-6) / 1e9,
                              "us_per_level_hop": us / (2 * plan.group_count)}))
        parts = torch.empty(D.NPARTS, dtype=torch.float64, device=dev)
        us = ev_time(lambda: D.spmv(kr.smap, kr.a, b, x, y, 1, x, parts), reps=50)
        print(json.dumps({"plan": name, "spmv_us": us, "gbs": spmv_bytes / (us * 1e-6) / 1e9}))
        for flags in (0,):
            f.sweep_flags = flags
            rhs = D.f64(bundle.rhs.data, dev)
            x0 = torch.zeros(m, dtype=torch.float64, device=dev)
            stop = P.StoppingCriteria(1e-8, 200)
            kr.solve(rhs, x0.clone(), stop)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = kr.solve(rhs, x0.clone(), stop)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(json.dumps({"plan": name, "flags": flags, "krylov_ms": dt * 1e3,
                              "its": res.iterations, "ms_per_it": dt * 1e3 / max(res.iterations, 0.5),
                              "launches": res.graph_launches}))


if __name__ == "__main__" and "--setup" not in sys.argv:
    main()


def setup_breakdown(dims=(100, 100, 100)):
    """Steady-state setup phases (second run), each bracketed by a sync."""
    from paper_2309_11488_b200.analysis import permute_device
    bundle = P.generate(P.GeneratorSpec(*dims, seed=0))
    a = bundle.a
    bsr = D.DevBSR.upload(a)
    out = {}
    for rep in range(2):
        for name, backend in (("level", P.Backend.LEVEL_SCHEDULED),
                              ("color", P.Backend.GRAPH_COLORED)):
            t = {}

            def mark(key, t0=[time.perf_counter()]):
                torch.cuda.synchronize()
                now = time.perf_counter()
                t[key] = (now - t0[0]) * 1e3
                t0[0] = now
            mark("start")
            D.find_diagonal(bsr.pat); mark("find_diag")
            g, ng = D.groups(bsr.pat, "level" if name == "level" else "color"); mark("groups")
            plan = P.analysis._device_plan(P.Strategy.LEVEL_SCHEDULING, g, bsr.pat.n, ng); mark("plan_sort")
            ap = permute_device(bsr, plan); mark("permute")
            lu = D.DevBSR(ap.pat, 3, ap.vals.clone()); mark("clone")
            diag = D.find_diagonal(lu.pat); mark("find_diag2")
            smap = plan.slice_map(); mark("slice_map")
            f = factor_device(a, plan, bsr); mark("factor_device_total")
            kr = DeviceKrylov.build(a, f, f._a_perm); mark("operator_sell")
            if rep == 1:
                print(json.dumps({"setup_breakdown": name, **{k: round(v, 3) for k, v in t.items()}}))


if __name__ == "__main__" and "--setup" in sys.argv:
    setup_breakdown()
