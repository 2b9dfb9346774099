#!/usr/bin/env python
"""Benchmark: ILU0-BiCGStab solve of the 1M-cell 3x3-block system (BASELINE C4).

One step = one complete solve as ``solve_with_fallback`` performs it (device
analysis -> permutation -> ILU0 factorisation -> operator layout ->
BiCGStab to tol 1e-8) on ``generate(GeneratorSpec(100,100,100, seed=0))``
(draw-for-draw the reference generator).  With N ranks the global grid is
100 x 100 x 100N, each GPU owns a contiguous 1M-cell z-slab (weak scaling),
the preconditioner is block-Jacobi ILU0 per slab and SpMV exchanges halos.

  value     cells solved per second, all ranks (Mcells/s = total cells / solve
            time), inputs resident in HBM, CUDA events, max over ranks;
  e2e       the same metric through the drop-in API ``solve_with_fallback``
            with HOST numpy buffers (matrix + rhs H2D, solution D2H timed);
  roofline  the dominant kernel's algorithmic bytes / its CUDA-event time vs
            MEASURED_PEAKS.json hbm_gbs (bytes per unit in DESIGN.md §4);
  cpu_baseline  the oracle port (numpy restatement of the reference) on a
            bounded slab of the same generator, 1 host core.

``--impl reference`` times that CPU port alone (rank 0) on the same metric,
with every host core: one independent slab solve per core per step (the
reference solves a system single-threaded and runs independent systems
concurrently).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ILU0-BiCGStab solve ms & iters/sec at 1M cells; SpMV/trsv HBM GB/s vs peak"
UNIT = "Mcells/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", default="100,100,100", help="cells per GPU (nx,ny,nz)")
    ap.add_argument("--backend", default="color", choices=["level", "color"])
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--boost", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--wells", type=int, default=20,
                    help="standard wells of the extra wells run (0: skip it)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-full", action="store_true",
                    help="skip the single-core full-workload port solve in cpu_baseline")
    ap.add_argument("--no-other-plan", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--ref-slab", type=int, default=2, help="z-planes of the CPU sample")
    ap.add_argument("--force-dist", action="store_true",
                    help="take the multi-GPU code path even with one rank (smoke test)")
    ap.add_argument("--dist-comm", default="mesh", choices=["mesh", "nccl"],
                    help="N>1: peer-memory device loop (default) or NCCL host loop")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """SM clock and clock-event reasons sampled across the timed region: NVML
    every 10 ms from a thread (at least one sample however short the region),
    else ``nvidia-smi -lms 100`` (whose first sample can come after a short
    region has ended)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    BITS = (0x8, 0x40, 0x20, 0x4)   # nvmlClocksEventReason{Hw,HwThermal,SwThermal}Slowdown, SwPowerCap

    def __init__(self, index=0):
        self.index, self.proc, self.out = index, None, None
        self.period = float(os.environ.get("B2S_CLOCK_MS", "10")) / 1e3
        self.nvml = self.handle = None
        try:
            import pynvml as N
            N.nvmlInit()
            try:   # the CUDA ordinal's PCI address (CUDA_VISIBLE_DEVICES may renumber)
                import torch
                pr = torch.cuda.get_device_properties(index)
                bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
                self.handle = N.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.handle = N.nvmlDeviceGetHandleByIndex(index)
            self.nvml = N
        except Exception:
            self.nvml = None

    def _loop(self):
        N = self.nvml
        while True:
            try:
                self.samples.append((N.nvmlDeviceGetClockInfo(self.handle, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetMaxClockInfo(self.handle, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetCurrentClocksEventReasons(self.handle)))
            except Exception:
                pass
            if self.done.wait(self.period):
                break

    def start(self):
        if self.nvml is not None:
            import threading
            self.samples, self.done = [], threading.Event()
            self.thread = threading.Thread(target=self._loop, daemon=True)
            self.thread.start()
            return
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.out, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.nvml is not None:
            self.done.set()
            self.thread.join(timeout=5)
            sm = sorted(float(r[0]) for r in self.samples)
            reasons = sorted({n for r in self.samples for n, b in zip(self.NAMES, self.BITS)
                              if r[2] & b})
            return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                    "sm_max_mhz": max(float(r[1]) for r in self.samples) if sm else None,
                    "reasons": reasons, "samples": len(sm), "sampler": "nvml 10 ms"}
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        rows = []
        try:
            self.out.flush()
            self.out.seek(0)
            rows = [[c.strip() for c in ln.split(",")] for ln in self.out.read().splitlines()
                    if ln.strip()]
        except Exception:
            pass
        rows = [r for r in rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        sm = sorted(float(r[0]) for r in rows)
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm),
                "sampler": "nvidia-smi 100 ms"}


# ---------------------------------------------------------------------------
# CPU port: cpu_baseline and --impl reference

def host_info():
    """Cores and CPU model of the host the CPU baseline runs on."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": model}


def cpu_port_sample(args, nx, ny, slab, per_op=False):
    """Single-core CPU solve of a bounded slab of the workload: the unmodified
    reference (baseline/_ref) when installed, else the oracle port; with
    ``per_op`` also SURVEY 8(d)'s per-op times on the same sample."""
    bs = reference_module()
    if bs is None:
        return _port_sample(args, nx, ny, slab, per_op)
    g = bs.generate(bs.GeneratorSpec(nx, ny, slab, seed=0, diagonal_boost=args.boost))
    a, rhs = g.a, g.rhs
    cfg = bs.SolverConfig(backend=bs.Backend(args.backend), stop=bs.StoppingCriteria(args.tol, 200))
    t0 = time.perf_counter()
    _, rep = bs.solve_with_fallback(cfg, a, rhs)
    dt = time.perf_counter() - t0
    cells = a.num_block_rows
    out = {"seconds": dt, "cells": cells, "iterations": rep.iterations, "kind": "reference",
           "value": cells / dt / 1e6,
           "sample": f"unmodified reference solve_with_fallback ({args.backend} plan + ILU0 + "
                     f"BiCGStab to tol {args.tol:g}) of GeneratorSpec({nx},{ny},{slab},seed=0): "
                     f"{cells} cells, {rep.iterations} its, {dt:.2f} s, 1 core"}
    if per_op:
        def t(fn):
            t1 = time.perf_counter()
            res = fn()
            return res, (time.perf_counter() - t1) * 1e3
        plan, t_plan = t(lambda: (bs.level_schedule if args.backend == "level"
                                  else bs.graph_color)(a.pattern))
        f, t_fact = t(lambda: bs.decompose(a, plan))
        _, t_spmv = t(lambda: bs.spmv(a, rhs))
        _, t_apply = t(lambda: f.apply_array(rhs.data))
        out["per_op_ms"] = {"plan": t_plan, "decompose": t_fact, "spmv": t_spmv,
                            "ilu0_apply": t_apply}
    return out


def _port_sample(args, nx, ny, slab, per_op=False):
    from oracle import port as O
    from paper_2309_11488_b200.synthetic import GeneratorSpec, generate
    g = generate(GeneratorSpec(nx, ny, slab, seed=0, diagonal_boost=args.boost))
    a = g.a
    rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
    t0 = time.perf_counter()
    x, rep, groups, fb = O.solve(rp, ci, v3, g.rhs.data, args.backend, args.tol)
    dt = time.perf_counter() - t0
    cells = a.num_block_rows
    out = {"seconds": dt, "cells": cells, "iterations": rep.iterations, "kind": "port",
           "value": cells / dt / 1e6,
           "sample": f"oracle port full solve ({args.backend} plan + ILU0 + BiCGStab to tol "
                     f"{args.tol:g}) of GeneratorSpec({nx},{ny},{slab},seed=0): {cells} cells, "
                     f"{rep.iterations} its, {dt:.2f} s, 1 core"}
    if per_op:   # the reference's per-op costs on the same sample (ms)
        def t(fn):
            t1 = time.perf_counter()
            res = fn()
            return res, (time.perf_counter() - t1) * 1e3
        grp, t_plan = t(lambda: (O.level_groups if args.backend == "level" else O.color_groups)(rp, ci))
        plan = O.plan_from_groups(grp)
        f, t_fact = t(lambda: O.ilu0(rp, ci, v3, plan))
        _, t_spmv = t(lambda: O.spmv(rp, ci, v3, g.rhs.data))
        _, t_apply = t(lambda: O.ilu0_apply(f, g.rhs.data))
        out["per_op_ms"] = {"plan": t_plan, "decompose": t_fact, "spmv": t_spmv,
                            "ilu0_apply": t_apply}
    return out


def full_port_solve(args, nx, ny, nz):
    """One single-core oracle-port solve of the whole workload (pins the
    per-cell extrapolation of the slab samples; ~45 s at C4)."""
    s = _port_sample(args, nx, ny, nz)
    return {"value": s["value"], "unit": UNIT, "seconds": s["seconds"],
            "iterations": s["iterations"], "cores": 1, "kind": "port", "sample": s["sample"]}


# ---------------------------------------------------------------------------
# reference arm: the UNMODIFIED reference (baseline/_ref) on the host cores

REF_DIR = ROOT / "baseline" / "_ref"
_SLABS: list = []          # per-worker slab systems, set before the pool forks


def reference_module():
    """``blocksolve`` from baseline/_ref (pip --target install of the
    unmodified /root/reference/pkg), or None when absent."""
    if not (REF_DIR / "blocksolve").is_dir():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import blocksolve
    return blocksolve


def c4_slabs(nx, ny, nz, boost, parts, bs=None):
    """Generate the C4 system (the reference's own generator when available;
    ours is draw-for-draw identical) and cut it into ``parts`` contiguous
    z-slabs: each slab's diagonal block (couplings to other slabs dropped,
    the paper's MPI block-Jacobi decomposition) and its rhs rows."""
    import numpy as np
    if bs is not None:
        g = bs.generate(bs.GeneratorSpec(nx, ny, nz, seed=0, diagonal_boost=boost))
    else:
        from paper_2309_11488_b200.synthetic import GeneratorSpec, generate
        g = generate(GeneratorSpec(nx, ny, nz, seed=0, diagonal_boost=boost))
    rp, ci = g.a.pattern.row_pointers, g.a.pattern.column_indices
    v3 = g.a.as_block_row_major().values.reshape(-1, 3, 3)
    rhs = g.rhs.data
    plane = nx * ny
    bounds = np.linspace(0, nz, parts + 1).round().astype(int)
    slabs = []
    for z0, z1 in zip(bounds[:-1], bounds[1:]):
        r0, r1 = z0 * plane, z1 * plane
        lo, hi = int(rp[r0]), int(rp[r1])
        cols = ci[lo:hi]
        keep = (cols >= r0) & (cols < r1)
        rows = np.repeat(np.arange(r1 - r0), np.diff(rp[r0:r1 + 1]))
        srp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows[keep], minlength=r1 - r0), out=srp[1:])
        slabs.append((srp, (cols[keep] - r0).astype(np.int64),
                      np.ascontiguousarray(v3[lo:hi][keep]).reshape(-1),
                      rhs[3 * r0:3 * r1].copy()))
    return slabs, rp.size - 1


def _ref_slab_solve(task):
    """One slab solve by the unmodified reference's solve_with_fallback (or
    the oracle port when the reference is not installed)."""
    k, backend, tol = task
    rp, ci, vals, rhs = _SLABS[k]
    bs = reference_module()
    t0 = time.perf_counter()
    if bs is not None:
        a = bs.BlockMatrix(bs.SparsityPattern(rp.size - 1, rp, ci), 3, vals)
        b = bs.BlockVector(rhs, 3)
        t0 = time.perf_counter()
        cfg = bs.SolverConfig(backend=bs.Backend(backend), stop=bs.StoppingCriteria(tol, 200))
        _, rep = bs.solve_with_fallback(cfg, a, b)
        its, conv = rep.iterations, rep.converged
    else:
        from oracle import port as O
        _, rep, _, _ = O.solve(rp, ci, vals.reshape(-1, 3, 3), rhs, backend, tol)
        its, conv = rep.iterations, rep.converged
    return {"cells": rp.size - 1, "seconds": time.perf_counter() - t0, "iterations": its,
            "converged": bool(conv)}


def run_reference(args):
    """The reference's own CPU path on the host, every core: each step solves
    the full C4 workload (1,000,000 cells) as ``W`` contiguous z-slab systems
    (C4's diagonal blocks, one per core, the paper's MPI-style block-Jacobi
    decomposition), each by the UNMODIFIED reference ``solve_with_fallback``
    single-threaded (baseline/_ref); value = cells / the step's wall time.
    Rank 0 only (the other ranks exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    import multiprocessing
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    nx, ny, nz = (int(v) for v in args.grid.split(","))
    workers = max(1, min(os.cpu_count() or 1, int(os.environ.get("B2S_REF_WORKERS", "64")), nz))
    bs = reference_module()
    kind = "reference" if bs is not None else "port"
    slabs, cells = c4_slabs(nx, ny, nz, args.boost, workers, bs)
    _SLABS[:] = slabs
    tasks = [(k, args.backend, args.tol) for k in range(len(slabs))]
    rounds = []
    with multiprocessing.get_context("fork").Pool(workers) as pool:
        for _ in range(args.warmup):
            pool.map(_ref_slab_solve, tasks, chunksize=1)
        for _ in range(args.steps):
            t0 = time.perf_counter()
            res = pool.map(_ref_slab_solve, tasks, chunksize=1)
            rounds.append((time.perf_counter() - t0, res))
    secs = sum(r[0] for r in rounds)
    value = cells * len(rounds) / secs / 1e6
    last = rounds[-1][1]
    its = sorted({r["iterations"] for r in last})
    per_slab = sum(r["seconds"] for r in last) / len(last)
    sample = (f"{'unmodified reference (baseline/_ref) solve_with_fallback' if bs else 'oracle port'}"
              f" ({args.backend} plan + ILU0 + BiCGStab to tol {args.tol:g}) of each of "
              f"{len(slabs)} z-slab diagonal blocks of C4 GeneratorSpec({nx},{ny},{nz},seed=0), "
              f"{cells} cells per step, one process per core; slab iterations {its}, "
              f"{per_slab:.1f} s per slab solve")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * secs / len(rounds),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 0)",
            "config": bench_config(args, nx, ny, nz, cells),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind,
                             "sample": sample,
                             "single_core_value": cells / per_slab / len(slabs) / 1e6,
                             "all_converged": all(r["converged"] for _, rr in rounds for r in rr),
                             "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_config(args, nx, ny, nz, cells):
    """The workload both arms run (identical dict: same_config)."""
    return {"workload": f"C4 GeneratorSpec({nx},{ny},{nz},seed=0): {cells} cells, 3x3 blocks, "
                        f"full solve (plan+permute+ILU0+BiCGStab) to tol {args.tol:g}",
            "backend": args.backend, "tol": args.tol, "cells_per_gpu": cells,
            "block_size": 3, "boost": args.boost}


def count_step_kernels(fn):
    """Kernels one step launches, counted by the CUDA profiler (CUPTI)."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"
                 and not e.name.startswith("Memcpy") and not e.name.startswith("Memset")]
    except Exception:
        return None
    ours = sum(1 for n in names if "b2s::" in n)
    cub = sum(1 for n in names if "cub::" in n)
    return {"per_step": ours + cub, "b2s": ours, "cub": cub, "other": len(names) - ours - cub}


# ---------------------------------------------------------------------------

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.force_dist:
        if "RANK" not in os.environ:   # --force-dist without a launcher: a world of one
            os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0",
                               "MASTER_ADDR": "127.0.0.1",
                               "MASTER_PORT": os.environ.get("MASTER_PORT", "29517")})
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from bench_dist import run_distributed
        return run_distributed(args, world, rank, local, METRIC, UNIT, Clocks, peaks,
                               cpu_port_sample, count_step_kernels)
    run_single(args)


def run_single(args):
    import numpy as np
    import torch

    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200 import _device as D
    from paper_2309_11488_b200.bridge import DeviceSolver

    dev = torch.device("cuda", torch.cuda.current_device())
    nx, ny, nz = (int(v) for v in args.grid.split(","))
    stop = P.StoppingCriteria(args.tol, 200)
    bundle = P.generate(P.GeneratorSpec(nx, ny, nz, seed=0, diagonal_boost=args.boost))
    a, rhs = bundle.a, bundle.rhs
    n, b = a.num_block_rows, a.block_size
    nnz = a.pattern.num_blocks
    bsr = D.DevBSR.upload(a)
    rhs_d = D.f64(rhs.data, dev)
    x_d = torch.zeros(n * b, dtype=torch.float64, device=dev)
    st = torch.cuda.current_stream()

    def measure(backend_name, steps, warmup, clocks=None, wells=None):
        cfg = P.SolverConfig(backend=P.Backend.from_name(backend_name), stop=stop)
        out = {}

        def step():
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            # nothing derived from the pattern survives between steps (the
            # diagonal positions are otherwise cached on the uploaded pattern)
            bsr.pat.__dict__.pop("_diag", None)
            e0.record(st)
            solver = DeviceSolver(a, bsr, cfg, wells=wells).setup()
            e1.record(st)
            x_d.zero_()
            res = solver.solve(rhs_d, x_d, stop, x0_zero=True)   # x_d was zeroed
            e2.record(st)
            return solver, res, (e0, e1, e2)
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        # no cyclic-GC pass inside the timed region (a pass over the host
        # heap stalls the thread that feeds the device loop for milliseconds)
        gc.collect()
        gc.disable()
        if clocks:
            clocks.start()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its, launches, evs = [], 0, []
        t0.record(st)
        solver = None
        for _ in range(steps):
            solver = None   # each step is a fresh setup: free the previous one first
            solver, res, ev = step()
            its.append(float(res.iterations))
            launches += int(res.graph_launches) * int(res.kernels_per_iteration)
            evs.append(ev)
        t1.record(st)
        torch.cuda.synchronize()
        gc.enable()
        if clocks:
            out["clocks"] = clocks.stop()
        ms = t0.elapsed_time(t1) / steps
        per = [e[0].elapsed_time(e[2]) for e in evs]
        out["step_ms_min_max"] = [min(per), max(per)]
        out.update({
            "solve_ms": ms, "iterations": sum(its) / len(its),
            "setup_ms": sum(e[0].elapsed_time(e[1]) for e in evs) / steps,
            "krylov_ms": sum(e[1].elapsed_time(e[2]) for e in evs) / steps,
            "groups": solver.plan.group_count, "gpu_launches": launches,
            "converged": bool(res.converged)})
        out["iters_per_s"] = out["iterations"] / (out["krylov_ms"] / 1e3)
        out["solver"] = solver
        return out

    clocks = Clocks(torch.cuda.current_device())
    main_run = measure(args.backend, args.steps, args.warmup, clocks)
    other = None
    if not args.no_other_plan:
        oname = "level" if args.backend == "color" else "color"
        other = measure(oname, max(3, args.steps // 2), 2)
        other.pop("solver")
        other["backend"] = oname

    # ---- the same system with separately applied standard wells (SURVEY
    # 8(f) row 1): the well terms run inside the device loop
    wells_run = None
    if args.wells > 0:
        wg = P.generate(P.GeneratorSpec(nx, ny, nz, seed=0, diagonal_boost=args.boost,
                                        well_count=args.wells, well_depth=min(nz, 10)))
        assert np.array_equal(wg.a.values, a.values)   # the wells are drawn after A and b
        wells_run = measure(args.backend, max(3, args.steps // 2), 2, wells=wg.wells)
        wells_run.pop("solver")
        wells_run.update({"wells": args.wells, "kind": "standard", "perforations_per_well":
                          min(nz, 10)})

    # ---- per-kernel CUDA-event timing on the headline solver's data
    solver = main_run.pop("solver")
    f, kr = solver.fact, solver.krylov
    m = n * b
    xp = torch.rand(m, dtype=torch.float64, device=dev)
    yp = torch.empty(m, dtype=torch.float64, device=dev)
    zp = torch.empty(m, dtype=torch.float64, device=dev)
    parts = torch.empty(D.NPARTS, dtype=torch.float64, device=dev)

    def timed(fn, reps=args.kernel_reps):
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
    t_apply = timed(lambda: f.apply_device(xp, zp))
    spmv_bytes = nnz * 76 + (n + 1) * 4 + 48 * n
    if f.phased:
        # phased sweeps (colourings): no sentinel fills; the intermediate y of
        # a 2-group plan is never stored, so the kernel's own minimum is r in,
        # z out (48 B/row) instead of SURVEY §8(d)'s r->y->z (96 B/row)
        t_sweeps = t_apply
        apply_bytes = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + \
            (48 if f.plan.group_count == 2 else 96) * n
    else:
        t_fill = timed(lambda: (D.fill_sentinel(yp, m), D.fill_sentinel(zp, m)))
        t_sweeps = max(t_apply - t_fill, 1e-3)
        apply_bytes = (nnz - n) * 76 + 72 * n + 8 * (n + 1) + 96 * n
    hbm, peak_kind = peaks()
    spmv_gbs = spmv_bytes / (t_spmv * 1e-6) / 1e9
    apply_gbs = apply_bytes / (t_sweeps * 1e-6) / 1e9
    dom = ("ilu0_apply (fwd+bwd sweeps)", apply_gbs, apply_bytes, t_sweeps) \
        if t_sweeps >= t_spmv else ("bsr_spmv", spmv_gbs, spmv_bytes, t_spmv)
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get(f"{args.backend}:{dom[0]}")
        except Exception:
            traffic = None

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        cfg = P.SolverConfig(backend=P.Backend.from_name(args.backend), stop=stop)
        # the assembler's output buffers are page-locked host memory (allocated
        # once, outside the timed region); every step copies them H2D inside it
        a_h, rhs_h = P.pin_host(a), P.pin_host(rhs)
        host_kind = "pinned" if D.is_pinned(torch.from_numpy(a_h.values)) else "pageable"
        for _ in range(2):
            xh, rep = P.solve_with_fallback(cfg, a_h, rhs_h)
        torch.cuda.synchronize()
        reps = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        e_conv = True
        for _ in range(reps):
            xh = None
            xh, rep = P.solve_with_fallback(cfg, a_h, rhs_h)
            e_conv &= rep.converged
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / reps
        # int64 row pointers / column indices (narrowed on the device), values, rhs
        h2d = (n + 1) * 8 + nnz * 8 + nnz * 72 + 24 * n
        e2e = {"value": n / dt / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 24 * n, "ms_per_step": dt * 1e3, "converged": e_conv,
               "host_memory": host_kind, "steps": reps}
        # the same call with ordinary (pageable) numpy arrays, as a caller that
        # did not allocate page-locked buffers hits it
        xh, rep = P.solve_with_fallback(cfg, a, rhs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            xh = None
            xh, rep = P.solve_with_fallback(cfg, a, rhs)
        torch.cuda.synchronize()
        dtp = (time.perf_counter() - t0) / reps
        e2e["pageable"] = {"value": n / dtp / 1e6, "ms_per_step": dtp * 1e3,
                           "converged": bool(rep.converged)}
        # a simulator's Newton loop: same pattern, new values every solve --
        # SolveSession analyses the pattern once (outside the timed region);
        # every step uploads values + rhs (page-locked), factorises, solves
        # and downloads x.  Reported beside e2e, not instead of it.
        sess = P.SolveSession(cfg, a_h.pattern, b)
        for _ in range(2):
            xh, rep = sess.solve(a_h, rhs_h)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s_conv = True
        for _ in range(reps):
            xh = None
            xh, rep = sess.solve(a_h, rhs_h)
            s_conv &= rep.converged
        torch.cuda.synchronize()
        dts = (time.perf_counter() - t0) / reps
        sess.close()
        e2e["values_refresh"] = {"value": n / dts / 1e6, "ms_per_step": dts * 1e3,
                                 "h2d_bytes_per_step": nnz * 72 + 24 * n,
                                 "d2h_bytes_per_step": 24 * n, "converged": s_conv,
                                 "api": "SolveSession.solve (pattern analysed once)"}

    cpu = None
    if not args.no_cpu:
        s = cpu_port_sample(args, nx, ny, args.ref_slab, per_op=True)
        cpu = {"value": s["value"], "unit": UNIT, "cores": 1, "kind": s["kind"],
               "sample": s["sample"], "per_op_ms": s["per_op_ms"], "host": host_info()}
        if not args.no_cpu_full:
            cpu["full_workload_single_core"] = full_port_solve(args, nx, ny, nz)

    clk = main_run.pop("clocks", None)
    launches = main_run.pop("gpu_launches")
    # measured kernel count of one step (CUPTI, outside the timed region):
    # every device kernel of setup + solve, ours (b2s::) and CUB's
    kinfo = count_step_kernels(lambda: DeviceSolver(a, bsr, P.SolverConfig(
        backend=P.Backend.from_name(args.backend), stop=stop)).setup().solve(
            rhs_d, torch.zeros_like(x_d), stop))
    if kinfo:
        launches = kinfo["per_step"] * args.steps
    line = {
        "metric": METRIC, "value": n / (main_run["solve_ms"] / 1e3) / 1e6, "unit": UNIT,
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": main_run["solve_ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seed 0)",
        "config": bench_config(args, nx, ny, nz, n),
        "nnzb_per_gpu": nnz, "parallelism": "single GPU",
        "l2": "inputs larger than L2 (579 MB matrix vs 126 MB)",
        **main_run,
        "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": dom[1], "peak": hbm,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": dom[1] / hbm,
                     "traffic": traffic, "algorithmic_bytes": dom[2], "us": dom[3],
                     "peak_note": "peak = the driver's copy bandwidth (b.copy_(a), half "
                                  "reads, half writes); these kernels are ~99% reads, "
                                  "which stream slightly faster, so frac can pass 1.0"},
        "kernels": {"spmv_us": t_spmv, "spmv_gbs": spmv_gbs, "spmv_frac": spmv_gbs / hbm,
                    "spmv_bytes": spmv_bytes, "ilu_apply_us": t_sweeps,
                    "ilu_apply_gbs": apply_gbs, "ilu_apply_frac": apply_gbs / hbm,
                    "ilu_apply_bytes": apply_bytes},
        "other_plan": other, "wells_run": wells_run, "clocks": clk, "e2e": e2e, "cpu_baseline": cpu,
        "gpu_launches": launches,
        "gpu_launches_per_step": kinfo,
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
