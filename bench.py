#!/usr/bin/env python
"""Benchmark: ILU0-BiCGStab solve on the 1M-cell 3x3-block system (BASELINE C4).

One step = one complete solve exactly as ``solve_with_fallback`` performs it
(device level schedule -> permutation -> ILU0 factorisation -> operator
layout -> BiCGStab to tol 1e-8), on ``generate(GeneratorSpec(100,100,100,
seed=0))`` (bit-identical to the reference generator).

  value  = cells x BiCGStab iterations / second, all ranks (Mcell-iter/s),
           inputs resident in HBM, CUDA-event timed (max over ranks);
  e2e    = the same metric through the public drop-in API
           ``solve_with_fallback(cfg, a, b)`` with HOST numpy buffers (matrix +
           rhs H2D and the solution D2H inside the timed region);
  roofline = the dominant kernel's algorithmic bytes / its CUDA-event time,
           against MEASURED_PEAKS.json hbm_gbs;
  cpu_baseline = the oracle port (a numpy restatement of the reference) on a
           bounded slab of the same generator, 1 host core.

``--impl reference`` times that CPU port alone (rank 0) on the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ILU0-BiCGStab solve ms & iters/sec at 1M cells; SpMV/trsv HBM GB/s vs peak"
UNIT = "Mcell-iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", default="100,100,100")
    ap.add_argument("--backend", default="level", choices=["level", "color"])
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--boost", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--ref-slab", type=int, default=2, help="z-planes of the CPU sample")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index=0):
        self.samples = []
        self.index = index
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    self.samples.append([s.strip() for s in out.strip().split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 7
                          for i in range(4) if "Active" in s[3 + i]})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU port (the reference's algorithm restated in numpy): cpu_baseline + --impl reference

def cpu_port_sample(args, nx, ny, slab):
    from oracle import port as O
    from paper_2309_11488_b200.synthetic import GeneratorSpec, generate
    g = generate(GeneratorSpec(nx, ny, slab, seed=0, diagonal_boost=args.boost))
    a = g.a
    rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
    t0 = time.perf_counter()
    x, rep, groups, fb = O.solve(rp, ci, v3, g.rhs.data, args.backend, args.tol)
    dt = time.perf_counter() - t0
    cells = a.num_block_rows
    return {"seconds": dt, "cells": cells, "iterations": rep.iterations,
            "value": cells * rep.iterations / dt / 1e6,
            "sample": f"oracle port full solve (plan+ILU0+BiCGStab tol {args.tol:g}) of "
                      f"GeneratorSpec({nx},{ny},{slab},seed=0), {cells} cells, "
                      f"{rep.iterations} its, {dt:.2f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nx, ny, nz = (int(v) for v in args.grid.split(","))
    for _ in range(args.warmup):
        cpu_port_sample(args, nx, ny, args.ref_slab)
    times, vals, last = [], [], None
    for _ in range(args.steps):
        last = cpu_port_sample(args, nx, ny, args.ref_slab)
        times.append(last["seconds"])
        vals.append(last["value"])
    value = sum(vals) / len(vals)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C4 GeneratorSpec({nx},{ny},{nz},seed=0) sampled as a "
                                   f"{args.ref_slab}-plane slab", "backend": args.backend,
                       "tol": args.tol, "block_size": 3},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": last["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200 import _device as D
    from paper_2309_11488_b200.bridge import DeviceSolver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    nx, ny, nz = (int(v) for v in args.grid.split(","))
    backend = P.Backend.from_name(args.backend)
    stop = P.StoppingCriteria(args.tol, 200)
    cfg = P.SolverConfig(backend=backend, stop=stop)

    bundle = P.generate(P.GeneratorSpec(nx, ny, nz, seed=0, diagonal_boost=args.boost))
    a, rhs = bundle.a, bundle.rhs
    n, b = a.num_block_rows, a.block_size
    nnz = a.pattern.num_blocks
    bsr = D.DevBSR.upload(a)
    rhs_d = D.f64(rhs.data, dev)
    x_d = torch.zeros(n * b, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()

    def step():
        solver = DeviceSolver(a, bsr, cfg).setup()
        x_d.zero_()
        res = solver.solve(rhs_d, x_d, stop)
        return solver, res

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        solver, res = step()
    barrier()
    clocks = Clocks(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = []
    launches = 0
    e0.record(st)
    for _ in range(args.steps):
        solver, res = step()
        its.append(float(res.iterations))
        launches += int(res.graph_launches) * int(res.kernels_per_iteration)
    e1.record(st)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    iters = sum(its) / len(its)
    value = world * n * iters / (ms_step / 1e3) / 1e6

    # ---- per-kernel CUDA-event timing on the same data (the roofline)
    f = solver.fact
    kr = solver.krylov
    m = n * b
    xp = torch.rand(m, dtype=torch.float64, device=dev)
    yp = torch.empty(m, dtype=torch.float64, device=dev)
    parts = torch.empty(D.NPARTS, dtype=torch.float64, device=dev)
    reps = args.kernel_reps

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        for _ in range(reps):
            fn()
        s1.record(st)
        torch.cuda.synchronize()
        return s0.elapsed_time(s1) / reps * 1e3   # us

    t_spmv = timed(lambda: D.spmv(kr.smap, kr.a, b, xp, yp, 1, xp, parts))
    zout = torch.empty(m, dtype=torch.float64, device=dev)
    t_apply = timed(lambda: f.apply_device(xp, zout))
    # apply_device includes two sentinel fills; time them alone and subtract
    t_fill = timed(lambda: (D.fill_sentinel(yp, m), D.fill_sentinel(zout, m)))
    t_sweeps = max(t_apply - t_fill, 1e-3)
    spmv_bytes = nnz * 76 + (n + 1) * 4 + 48 * n
    apply_bytes = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 96 * n
    hbm, peak_kind = peaks()
    spmv_gbs = spmv_bytes / (t_spmv * 1e-6) / 1e9
    apply_gbs = apply_bytes / (t_sweeps * 1e-6) / 1e9
    # dominant kernel by share of an iteration (2 applies vs 2 SpMVs)
    dom = ("ilu0_apply (fwd+bwd sweeps)", apply_gbs, apply_bytes) if t_sweeps >= t_spmv \
        else ("bsr_spmv", spmv_gbs, spmv_bytes)
    prof = ROOT / "profiles" / "traffic.json"
    traffic = None
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(dom[0])
        except Exception:
            traffic = None

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        for _ in range(1):
            P.solve_with_fallback(cfg, a, rhs)
        torch.cuda.synchronize()
        reps_e2e = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        e_its = []
        for _ in range(reps_e2e):
            xh, rep = P.solve_with_fallback(cfg, a, rhs)
            e_its.append(rep.iterations)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps_e2e
        if world > 1:
            t = torch.tensor([dt], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = (n + 1) * 4 + nnz * 4 + nnz * 72 + 2 * 24 * n
        e2e = {"value": world * n * (sum(e_its) / len(e_its)) / dt / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 24 * n,
               "ms_per_step": dt * 1e3}

    cpu = None
    if rank == 0 and not args.no_cpu:
        s = cpu_port_sample(args, nx, ny, args.ref_slab)
        cpu = {"value": s["value"], "unit": UNIT, "cores": 1, "kind": "port",
               "sample": s["sample"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 0)",
            "config": {"workload": f"C4 GeneratorSpec({nx},{ny},{nz},seed=0), 3x3 blocks, "
                                   f"{n} cells/GPU, full solve (analysis+factor+BiCGStab) "
                                   f"to tol {args.tol:g}",
                       "backend": args.backend, "tol": args.tol, "cells_per_gpu": n,
                       "nnzb_per_gpu": nnz, "parallelism": f"replicas x{world}" if world > 1
                       else "single GPU", "l2": "inputs (579 MB matrix) larger than L2"},
            "iterations": iters, "solve_ms": ms_step, "iters_per_s": iters / (ms_step / 1e3),
            "setup_and_krylov": "per step",
            "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": dom[1], "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": dom[1] / hbm,
                         "traffic": traffic},
            "kernels": {"spmv_us": t_spmv, "spmv_gbs": spmv_gbs, "spmv_frac": spmv_gbs / hbm,
                        "spmv_bytes": spmv_bytes, "ilu_apply_us": t_sweeps,
                        "ilu_apply_gbs": apply_gbs, "ilu_apply_frac": apply_gbs / hbm,
                        "ilu_apply_bytes": apply_bytes, "levels": int(f.plan.group_count)},
            "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
