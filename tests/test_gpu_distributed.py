"""The partitioned (block-Jacobi slab) solver against the oracle, with all
shards in one process on one GPU (LocalComm).  The oracle is the reference's
own recipe for a partitioned preconditioner: drop_cross_blocks with the slab
partition -> decompose(level plan) -> bicgstab(full operator)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2309_11488_b200 as P  # noqa: E402
from oracle import port as O  # noqa: E402
from paper_2309_11488_b200.distributed import local_solver, slab_bounds, solve_shards  # noqa: E402


def oracle_partitioned(spec, world, tol):
    full = P.generate(spec)
    a = full.a
    rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
    nxy = spec.nx * spec.ny
    part = np.zeros(a.num_block_rows, dtype=np.int64)
    for r in range(world):
        z0, z1 = slab_bounds(spec.nz, world, r)
        part[z0 * nxy:z1 * nxy] = r
    jrp, jci, jv, _ = O.drop_cross(rp, ci, v3, part)
    f = O.ilu0(jrp, jci, jv, O.plan_from_groups(O.level_groups(jrp, jci)))
    x, rep = O.bicgstab(lambda v: O.spmv(rp, ci, v3, v), lambda r: O.ilu0_apply(f, r),
                        full.rhs.data, tol=tol)
    return x, rep


@pytest.mark.parametrize("dims,world", [((8, 7, 12), 2), ((6, 6, 9), 3), ((10, 8, 8), 4)])
def test_sharded_solve_matches_partitioned_oracle(dims, world):
    spec = P.GeneratorSpec(*dims, seed=5, diagonal_boost=1e-2)
    tol = 1e-8
    xo, ro = oracle_partitioned(spec, world, tol)
    shards, comm = local_solver(spec, world)
    rep, xs = solve_shards(shards, comm, P.StoppingCriteria(tol, 200))
    x = np.concatenate([v.cpu().numpy() for v in xs])
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= 1.0, (rep.iterations, ro.iterations)
    assert np.linalg.norm(x - xo) <= 1e-6 * np.linalg.norm(xo)
    np.testing.assert_allclose(rep.initial_norm, ro.initial_norm, rtol=1e-12)


def test_one_shard_equals_single_gpu_solver():
    spec = P.GeneratorSpec(9, 8, 7, seed=2)
    shards, comm = local_solver(spec, 1)
    rep, xs = solve_shards(shards, comm, P.StoppingCriteria(1e-8, 200))
    b = P.generate(spec)
    x1, r1 = P.solve_with_fallback(P.SolverConfig(stop=P.StoppingCriteria(1e-8, 200)),
                                   b.a, b.rhs)
    assert rep.iterations == r1.iterations
    assert np.linalg.norm(xs[0].cpu().numpy() - x1.data) <= 1e-10 * np.linalg.norm(x1.data)
