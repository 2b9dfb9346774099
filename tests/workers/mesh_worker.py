"""One rank of a peer-memory sharded solve (tests/test_gpu_distributed.py).

Launched by torch.distributed.run with a gloo group (host rendezvous only:
the solve itself communicates through CUDA IPC peer memory).  Every rank
uses cuda:0 when --same-gpu is given, so two processes can exercise the IPC
path on a one-GPU box.  Rank 0 prints one JSON line.
"""
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    dims = tuple(int(v) for v in sys.argv[1].split(","))
    backend = sys.argv[2]
    same = "--same-gpu" in sys.argv
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0 if same else int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group("gloo")
    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200.distributed import (Shard, exchange_requests, generate_slab,
                                                   slab_bounds, solve_shard_mesh_dist)
    spec = P.GeneratorSpec(*dims, seed=5, diagonal_boost=1e-2)
    slab = generate_slab(spec, rank, world)
    owners = np.array([slab_bounds(spec.nz, world, r)[0] * spec.nx * spec.ny
                       for r in range(world)], dtype=np.int64)
    shard = Shard(slab, owners, P.Backend.from_name(backend))

    def gather(mine):
        out = [None] * world
        dist.all_gather_object(out, mine)
        return out
    exchange_requests([shard], world, gather)
    stop = P.StoppingCriteria(1e-8, 200)
    if "--fail-ipc-rank" in sys.argv:   # this rank cannot open its peers' buffers
        if rank == int(sys.argv[sys.argv.index("--fail-ipc-rank") + 1]):
            from paper_2309_11488_b200 import _device as D
            D.lib().b2s_ipc_open = lambda *args: 3
    from paper_2309_11488_b200.distributed import MeshUnavailable, NcclComm, solve_shards
    reps, xs, fallback = [], [], None
    for _ in range(2):
        if "--comm-loop" in sys.argv or fallback:   # the host-driven loop
            rep, xv = solve_shards([shard], NcclComm(shard), stop)
            x = xv[0]
        else:
            try:
                rep, x = solve_shard_mesh_dist(shard, stop, cache_key=backend)
            except MeshUnavailable as exc:   # every rank lands here alike
                fallback = str(exc)
                rep, xv = solve_shards([shard], NcclComm(shard), stop)
                x = xv[0]
        reps.append(rep)
        xs.append(x.cpu().numpy())
    allx = gather((rank, xs[0], xs[1]))
    if rank == 0:
        allx.sort(key=lambda t: t[0])
        x0 = np.concatenate([t[1] for t in allx])
        x1 = np.concatenate([t[2] for t in allx])
        print(json.dumps({"iterations": [r.iterations for r in reps],
                          "converged": [bool(r.converged) for r in reps],
                          "initial_norm": reps[0].initial_norm,
                          "rerun_bit_equal": bool(np.array_equal(x0, x1)),
                          "fallback": fallback,
                          "x": x0.tolist()}), flush=True)
    if getattr(shard, "mesh", None) is not None:
        shard.mesh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
