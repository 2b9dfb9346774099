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


def run_distributed(args, world, rank, local, metric, unit, Clocks, peaks, cpu_port_sample):
    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200.distributed import (NcclComm, Shard, exchange_requests,
                                                   generate_slab, slab_bounds,
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

    def e2e_step():                            # host slab in, host x out
        sh = Shard(slab, owners, backend)
        exchange_requests([sh], world, gather)
        if mesh:
            sh.mesh = shard.mesh                   # the IPC-shared buffers stay mapped
            rep, x = solve_shard_mesh_dist(sh, stop, cache_key=args.backend)
            x.cpu()
            return rep
        rep, xs = solve_shards([sh], NcclComm(sh), stop)
        xs[0].cpu()
        return rep
    e2e_ms, _ = (None, None) if args.no_e2e else timed(e2e_step, max(1, args.steps // 3), 1)
    n_total = spec.nx * spec.ny * spec.nz
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
            "iterations": iters, "solve_ms": ms, "clocks": clk,
            "e2e": None if e2e_ms is None else {
                "value": n_total / (e2e_ms / 1e3) / 1e6, "unit": unit, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": world * (slab.rp.size * 4 + slab.ci.size * 4
                                               + slab.vals3.size * 8 + slab.rhs.size * 8),
                "d2h_bytes_per_step": n_total * 24},
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
