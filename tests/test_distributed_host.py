"""Host-side logic of the multi-GPU path (no GPU): the slab generator is
draw-for-draw the full generator's rows, and the halo request routing works
across a world_size-2 gloo process group."""

import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp
from numpy.testing import assert_array_equal

from paper_2309_11488_b200.distributed import (HaloPlan, generate_slab, route_requests,
                                               slab_bounds)
from paper_2309_11488_b200.synthetic import GeneratorSpec, generate


@pytest.mark.parametrize("dims,world", [((6, 5, 8), 2), ((4, 3, 7), 3), ((5, 4, 6), 1),
                                        ((3, 3, 10), 4)])
def test_slab_rows_equal_full_generator(dims, world):
    spec = GeneratorSpec(*dims, seed=11, tz=0.3, diagonal_boost=0.7)
    full = generate(spec)
    rp, ci = full.a.pattern.row_pointers, full.a.pattern.column_indices
    v3 = full.a.values3d
    for r in range(world):
        s = generate_slab(spec, r, world)
        z0, z1 = slab_bounds(dims[2], world, r)
        assert (s.r0, s.r1) == (z0 * dims[0] * dims[1], z1 * dims[0] * dims[1])
        lo, hi = rp[s.r0], rp[s.r1]
        assert_array_equal(s.rp, rp[s.r0:s.r1 + 1] - lo)
        assert_array_equal(s.ci, ci[lo:hi])
        assert_array_equal(s.vals3, v3[lo:hi])
        assert_array_equal(s.rhs, full.rhs.data[s.r0 * 3:s.r1 * 3])


def test_slab_bounds_cover_the_grid():
    for nz in (1, 7, 100, 800):
        for world in (1, 2, 3, 8):
            if world > nz:
                continue
            b = [slab_bounds(nz, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == nz
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))


def test_halo_plan_stencil_ghosts():
    spec = GeneratorSpec(4, 3, 6, seed=1)
    s = generate_slab(spec, 1, 3)
    owners = np.array([slab_bounds(6, 3, r)[0] * 12 for r in range(3)])
    hp = HaloPlan(s, owners)
    # z-slab of 2 planes: ghosts are the plane below and the plane above
    assert_array_equal(hp.ghosts, np.r_[np.arange(12, 24), np.arange(48, 60)])
    assert set(hp.recv) == {0, 2}
    assert (hp.lcol[hp.own] < s.rows).all() and (hp.lcol[~hp.own] >= s.rows).all()


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec = GeneratorSpec(4, 3, 6, seed=1)
    slab = generate_slab(spec, rank, world)
    owners = np.array([slab_bounds(6, world, r)[0] * 12 for r in range(world)])
    hp = HaloPlan(slab, owners)

    def gather(mine):
        res = [None] * world
        dist.all_gather_object(res, mine)
        return res
    sends = route_requests([(rank, hp.requests())], gather)[rank]
    out[rank] = {h: v.tolist() for h, v in sends.items()}
    dist.barrier()
    dist.destroy_process_group()


def test_request_routing_over_gloo():
    world = 2
    port = 29000 + os.getpid() % 1000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    # rank 0 sends rank 1 its top plane, rank 1 sends rank 0 its bottom plane
    assert res[0] == {1: list(range(24, 36))}
    assert res[1] == {0: list(range(36, 48))}
