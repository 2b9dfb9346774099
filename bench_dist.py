"""Multi-GPU leg of bench.py (torchrun, one rank per GPU, NVLink peer memory).

Weak scaling: the global system is GeneratorSpec(nx, ny, nz * N, seed=0);
rank g owns z-planes [g*nz, (g+1)*nz) (1M cells at the default grid),
generated draw-for-draw as the rows of the global system.  One step = one
complete partitioned solve: per-slab level/colour plan + block-Jacobi ILU0
+ BiCGStab.  Default communication ("mesh"): every rank runs the
device-resident BiCGStab loop (one CUDA graph per iteration) and the kernels
talk to the peers through NVLink peer memory opened with CUDA IPC -- the
SpMV's ghost rows are read straight from the owners' vectors and the dot
products are all-reduced through per-rank mailboxes by the last CTA of each
reducing kernel (csrc/krylov.cu, b2s_mesh).  "--dist-comm nccl" runs the
host-driven loop with NCCL send/recv halos and all-reduces instead.  Times
are CUDA events on each rank, max over ranks.
"""

from __future__ import annotations

import json

import torch
import torch.distributed as dist


def kernel_roofline(shard, peaks):
    """Dominant kernels of the shard's iteration (SpMV over the owned rows with
    ghost columns, ILU0 application), CUDA-event timed on this rank, against
    SURVEY §8(d)'s algorithmic bytes for the shard (bench.py's formulas)."""
    from paper_2309_11488_b200 import _device as D
    n, b = shard.R, shard.b
    nnz = int(shard.slab.rp[-1])
    nloc = int(shard.pmat.pattern.num_blocks)
    m = n * b
    st = torch.cuda.current_stream()
    x = torch.rand((n + shard.G) * b, dtype=torch.float64, device=shard.dev)
    y = torch.empty(m, dtype=torch.float64, device=shard.dev)
    z = torch.empty(m, dtype=torch.float64, device=shard.dev)
    parts = torch.empty(D.NPARTS, dtype=torch.float64, device=shard.dev)

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    t_spmv = timed(lambda: D.spmv(shard.smap, shard.sell, b, x, y, 1, x, parts))
    t_apply = timed(lambda: shard.fact.apply_device(x[:m], z))
    spmv_bytes = nnz * 76 + (n + 1) * 4 + 48 * n
    apply_bytes = (nloc - n) * 76 + 72 * n + 8 * (n + 1) + \
        (48 if shard.plan.group_count == 2 else 96) * n
    hbm, kind = peaks()
    dom = (("ilu0_apply (fwd+bwd sweeps)", apply_bytes, t_apply) if t_apply >= t_spmv
           else ("bsr_spmv (halo columns)", spmv_bytes, t_spmv))
    gbs = dom[1] / (dom[2] * 1e-6) / 1e9
    return {"bound": "hbm", "kernel": dom[0], "achieved": gbs, "peak": hbm, "peak_kind": kind,
            "unit": "GB/s", "frac": gbs / hbm, "traffic": None, "algorithmic_bytes": dom[1],
            "us": dom[2], "spmv_us": t_spmv, "ilu_apply_us": t_apply}


def run_distributed(args, world, rank, local, metric, unit, Clocks, peaks, cpu_port_sample,
                    count_step_kernels=None):
    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200._lib import PeerTimeout
    from paper_2309_11488_b200.distributed import (MeshUnavailable, NcclComm, Shard,
                                                   exchange_requests, generate_slab, slab_bounds,
                                                   solve_shard_mesh_dist, solve_shards)
    import numpy as np

    nx, ny, nz = (int(v) for v in args.grid.split(","))
    spec = P.GeneratorSpec(nx, ny, nz * world, seed=0, diagonal_boost=args.boost)
    backend = P.Backend.from_name(args.backend)
    stop = P.StoppingCriteria(args.tol, 200)
    slab = generate_slab(spec, rank, world)
    owners = np.array([slab_bounds(spec.nz, world, r)[0] * nx * ny for r in range(world)],
                      dtype=np.int64)

    def gather(mine):
        out = [None] * world
        dist.all_gather_object(out, mine)
        return out

    st = torch.cuda.current_stream()
    mesh = getattr(args, "dist_comm", "mesh") == "mesh"
    shard = Shard(slab, owners, backend)       # matrix uploaded once (resident)
    exchange_requests([shard], world, gather)
    comm = None if mesh else NcclComm(shard)

    def step():
        shard.setup(backend)                   # plan + permute + ILU0 + layouts
        if mesh:
            return solve_shard_mesh_dist(shard, stop, cache_key=args.backend)[0]
        return solve_shards([shard], comm, stop)[0]

    # peer memory between these GPUs: if CUDA IPC / peer access is refused on
    # any rank (agreed on by all ranks: MeshUnavailable) or a peer times out,
    # the line is measured on the NCCL host loop and says so
    mesh_fallback = None
    if mesh:
        try:
            step()
        except (MeshUnavailable, PeerTimeout) as exc:
            mesh_fallback = f"{type(exc).__name__}: {exc}"[:300]
            if getattr(shard, "mesh", None) is not None:
                shard.mesh.close()
                shard.mesh = None
            mesh = False
            comm = NcclComm(shard)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = []
        e0.record(st)
        for _ in range(steps):
            its.append(fn().iterations)
        e1.record(st)
        torch.cuda.synchronize()
        dist.barrier()
        ms = torch.tensor([e0.elapsed_time(e1) / steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        return float(ms.item()), sum(its) / len(its)

    clocks = Clocks(local)
    clocks.start()
    ms, iters = timed(step, args.steps, args.warmup)
    clk = clocks.stop()

    # e2e, the single-GPU semantics: every step starts from HOST arrays --
    # each rank uploads its slab's pattern, block values and rhs from
    # page-locked buffers, re-plans the halo (host request routing + device
    # send lists), runs setup + solve, and reads its solution back into
    # page-locked memory.  (A values-only refresh of a resident pattern, the
    # next Newton step of a simulator, is reported beside it.)
    from paper_2309_11488_b200._device import pinned_copy
    from paper_2309_11488_b200.distributed import Slab
    ps = Slab(slab.rank, slab.world, slab.n_global, slab.r0, slab.r1, slab.b,
              pinned_copy(slab.rp), pinned_copy(slab.ci), pinned_copy(slab.vals3),
              pinned_copy(slab.rhs))
    x_h = torch.empty(slab.rows * slab.b, dtype=torch.float64, pin_memory=True)

    def e2e_step():
        sh = Shard(ps, owners, None)              # pattern + values H2D, halo plan
        exchange_requests([sh], world, gather)    # which rows every peer needs
        sh.rhs_d = torch.from_numpy(ps.rhs).to(sh.dev, non_blocking=True)   # rhs H2D
        sh.setup(backend)
        if mesh:
            rep, x = solve_shard_mesh_dist(sh, stop, cache_key=None)
        else:
            rep, xs = solve_shards([sh], NcclComm(sh), stop)
            x = xs[0]
        x_h.copy_(x, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if mesh:
            sh.mesh.close()
        return rep

    vals_h, rhs_h = ps.vals3.reshape(-1), ps.rhs

    def refresh_step():
        shard.refresh_values(vals_h, rhs_h)
        shard.setup(backend)
        if mesh:
            rep, x = solve_shard_mesh_dist(shard, stop, cache_key=args.backend)
        else:
            rep, xs = solve_shards([shard], comm, stop)
            x = xs[0]
        x_h.copy_(x, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return rep
    e2e_ms = ref_ms = None
    if not args.no_e2e:
        e2e_ms, _ = timed(e2e_step, max(1, args.steps // 3), 1)
        ref_ms, _ = timed(refresh_step, max(1, args.steps // 3), 1)
    n_total = spec.nx * spec.ny * spec.nz
    roof = kernel_roofline(shard, peaks)
    # kernels of one step on this rank (CUPTI), outside the timed region
    kinfo = count_step_kernels(step) if count_step_kernels else None
    cpu = None
    if rank == 0 and not args.no_cpu:   # same sample as the single-GPU line, rank 0 only
        smp = cpu_port_sample(args, nx, ny, args.ref_slab, per_op=True)
        cpu = {"value": smp["value"], "unit": unit, "cores": 1, "kind": smp["kind"],
               "sample": smp["sample"], "per_op_ms": smp["per_op_ms"]}
    if rank == 0:
        line = {
            "metric": metric, "value": n_total / (ms / 1e3) / 1e6, "unit": unit,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 0; per-rank slabs draw-for-draw)",
            "config": {"workload": f"C5 GeneratorSpec({nx},{ny},{nz}*{world},seed=0), "
                                   f"{slab.rows} cells/GPU z-slabs, block-Jacobi ILU0, halo "
                                   f"SpMV, all-reduced dots, tol {args.tol:g}",
                       "backend": args.backend, "cells_total": n_total,
                       "parallelism": f"slab x{world} ("
                                      + ("NVLink peer memory, device loop" if mesh else
                                         "NCCL, host loop") + ")"},
            "iterations": iters, "solve_ms": ms, "clocks": clk, "mesh_fallback": mesh_fallback,
            "e2e": None if e2e_ms is None else {
                "value": n_total / (e2e_ms / 1e3) / 1e6, "unit": unit, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": world * ((slab.rows + 1) * 8 + slab.ci.size * 8
                                               + slab.vals3.size * 8 + slab.rhs.size * 8),
                "d2h_bytes_per_step": n_total * 24, "host_memory": "pinned",
                "includes": "pattern + values + rhs upload, halo plan, setup, solve, x download",
                "values_only_refresh": {"value": n_total / (ref_ms / 1e3) / 1e6,
                                        "ms_per_step": ref_ms,
                                        "h2d_bytes_per_step": world * (slab.vals3.size * 8
                                                                       + slab.rhs.size * 8)}},
            "roofline": roof,
            "gpu_launches": (kinfo["per_step"] * args.steps * world) if kinfo else None,
            "gpu_launches_per_step": kinfo,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
