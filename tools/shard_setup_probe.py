"""Where a fresh shard's host setup goes (the N>1 e2e step of bench_dist.py
at one rank): cProfile of Shard() + exchange_requests + setup + a mesh solve.

python tools/shard_setup_probe.py
"""
import cProfile
import os
import pstats
import sys
import time
from pathlib import Path

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200._device import pinned_copy  # noqa: E402
from paper_2309_11488_b200.distributed import (Shard, Slab, exchange_requests,  # noqa: E402
                                               generate_slab, slab_bounds, solve_shards_mesh)

spec = P.GeneratorSpec(100, 100, 100, seed=0)
slab = generate_slab(spec, 0, 1)
ps = Slab(slab.rank, slab.world, slab.n_global, slab.r0, slab.r1, slab.b,
          pinned_copy(slab.rp), pinned_copy(slab.ci), pinned_copy(slab.vals3), pinned_copy(slab.rhs))
owners = np.array([0], dtype=np.int64)
stop = P.StoppingCriteria(1e-8, 200)


def step():
    sh = Shard(ps, owners, None)
    exchange_requests([sh], 1, lambda mine: [mine])
    sh.rhs_d = torch.from_numpy(ps.rhs).to(sh.dev, non_blocking=True)
    sh.setup(P.Backend.GRAPH_COLORED)
    rep, xs = solve_shards_mesh([sh], stop)
    torch.cuda.synchronize()
    return rep


for _ in range(2):
    step()
t0 = time.perf_counter()
step()
print("step ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
