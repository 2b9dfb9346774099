"""The partitioned (block-Jacobi slab) solver against the oracle, with all
shards in one process on one GPU (LocalComm).  The oracle is the reference's
own recipe for a partitioned preconditioner: drop_cross_blocks with the slab
partition -> decompose(level plan) -> bicgstab(full operator)."""

import numpy as np
import torch
import pytest

# (a hard per-test limit: a cross-shard wait that never resolves must fail the
# test, not hang the suite)
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300, method="thread")]

import paper_2309_11488_b200 as P  # noqa: E402
from oracle import port as O  # noqa: E402
from paper_2309_11488_b200.distributed import local_solver, slab_bounds, solve_shards  # noqa: E402


def oracle_partitioned(spec, world, tol, plan="level"):
    """The reference's partitioned recipe with the given plan (level schedule
    or graph colouring of the relaxed pattern)."""
    full = P.generate(spec)
    a = full.a
    rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
    nxy = spec.nx * spec.ny
    part = np.zeros(a.num_block_rows, dtype=np.int64)
    for r in range(world):
        z0, z1 = slab_bounds(spec.nz, world, r)
        part[z0 * nxy:z1 * nxy] = r
    jrp, jci, jv, _ = O.drop_cross(rp, ci, v3, part)
    groups = (O.level_groups if plan == "level" else O.color_groups)(jrp, jci)
    f = O.ilu0(jrp, jci, jv, O.plan_from_groups(groups))
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


@pytest.mark.parametrize("dims,world,backend",
                         [((8, 7, 12), 2, "level"), ((6, 6, 9), 3, "color"),
                          ((10, 8, 8), 4, "level"), ((12, 10, 16), 4, "color")])
def test_mesh_solve_matches_partitioned_oracle(dims, world, backend):
    """The peer-memory device loop (csrc/krylov.cu b2s_mesh: ghost rows read
    from the owners' vectors, mailbox all-reduce in the control CTA), all
    shards on one GPU, each on its own stream and host thread."""
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    spec = P.GeneratorSpec(*dims, seed=5, diagonal_boost=1e-2)
    tol = 1e-8
    be = P.Backend.from_name(backend)
    shards, comm = local_solver(spec, world, be)
    rep_h, xs_h = solve_shards(shards, comm, P.StoppingCriteria(tol, 200))
    rep, xs = solve_shards_mesh(shards, P.StoppingCriteria(tol, 200))
    x = np.concatenate([v.cpu().numpy() for v in xs])
    xh = np.concatenate([v.cpu().numpy() for v in xs_h])
    assert rep.converged and rep_h.converged
    # partitioned solves: the north star's band is +-10% (rounding-level
    # differences in the dot products move ill-conditioned cases by a few)
    assert abs(rep.iterations - rep_h.iterations) <= max(1.0, 0.1 * rep_h.iterations), \
        (rep.iterations, rep_h.iterations)
    np.testing.assert_allclose(rep.initial_norm, rep_h.initial_norm, rtol=1e-12)
    assert np.linalg.norm(x - xh) <= 1e-6 * np.linalg.norm(xh)
    # against the reference's partitioned recipe with the same plan
    xo, ro = oracle_partitioned(spec, world, tol, backend)
    assert abs(rep.iterations - ro.iterations) <= max(1.0, 0.1 * ro.iterations), \
        (rep.iterations, ro.iterations)
    assert np.linalg.norm(x - xo) <= 1e-6 * np.linalg.norm(xo)
    # a second solve on the same buffers (sequence numbers move on)
    rep2, xs2 = solve_shards_mesh(shards, P.StoppingCriteria(tol, 200))
    assert rep2.iterations == rep.iterations
    assert np.array_equal(np.concatenate([v.cpu().numpy() for v in xs2]), x)


def test_mesh_one_shard_equals_single_gpu_solver():
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    spec = P.GeneratorSpec(9, 8, 7, seed=2)
    shards, _ = local_solver(spec, 1)
    rep, xs = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    b = P.generate(spec)
    x1, r1 = P.solve_with_fallback(P.SolverConfig(stop=P.StoppingCriteria(1e-8, 200)),
                                   b.a, b.rhs)
    assert rep.iterations == r1.iterations
    assert np.linalg.norm(xs[0].cpu().numpy() - x1.data) <= 1e-10 * np.linalg.norm(x1.data)


def test_mesh_two_processes_over_ipc(tmp_path):
    """Two processes, one shard each, peer buffers opened through CUDA IPC
    (the multi-GPU path of bench.py; both ranks on cuda:0 here)."""
    import json
    import socket
    import subprocess
    import sys
    from pathlib import Path

    from paper_2309_11488_b200.distributed import solve_shards_mesh
    dims, world = (8, 7, 12), 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(root / "tests" / "workers" / "mesh_worker.py"), "8,7,12", "level", "--same-gpu"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    got = json.loads(line)
    spec = P.GeneratorSpec(*dims, seed=5, diagonal_boost=1e-2)
    shards, _ = local_solver(spec, world, P.Backend.LEVEL_SCHEDULED)
    rep, xs = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    x = np.concatenate([v.cpu().numpy() for v in xs])
    assert all(got["converged"]) and got["rerun_bit_equal"]
    assert got["iterations"][0] == rep.iterations
    assert np.array_equal(np.asarray(got["x"]), x)   # same kernels, same sums: same bits


def test_refresh_values_equals_fresh_shard():
    """A shard refreshed with new values (device gather of the owned blocks)
    solves exactly like a shard built from scratch with those values."""
    from paper_2309_11488_b200.distributed import Slab, solve_shards_mesh
    spec = P.GeneratorSpec(8, 7, 12, seed=5, diagonal_boost=1e-2)
    shards, _ = local_solver(spec, 2, P.Backend.GRAPH_COLORED)
    rng = np.random.default_rng(3)
    fresh_slabs = []
    for s in shards:
        sl = s.slab
        v = sl.vals3 * (1.0 + 0.01 * rng.random(sl.vals3.shape))
        r = rng.uniform(-1, 1, sl.rhs.shape)
        fresh_slabs.append(Slab(sl.rank, sl.world, sl.n_global, sl.r0, sl.r1, sl.b, sl.rp, sl.ci,
                                v, r))
        s.refresh_values(v, r)
        s.setup(P.Backend.GRAPH_COLORED)
    rep1, xs1 = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    from paper_2309_11488_b200.distributed import Shard, exchange_requests
    owners = np.array([s.r0 for s in fresh_slabs], dtype=np.int64)
    fresh = [Shard(sl, owners, P.Backend.GRAPH_COLORED) for sl in fresh_slabs]
    exchange_requests(fresh, 2, lambda mine: [mine])
    rep2, xs2 = solve_shards_mesh(fresh, P.StoppingCriteria(1e-8, 200))
    assert rep1.iterations == rep2.iterations
    for a, b in zip(xs1, xs2):
        assert torch.equal(a, b)


def test_mesh_fused_colour_passes_match_unfused(monkeypatch):
    """2-colour shards: fused colour passes on the local block + ghost
    correction (b2s_mesh bnd_*) against the unfused mesh loop."""
    from paper_2309_11488_b200.distributed import _mesh_fused, solve_shards_mesh
    spec = P.GeneratorSpec(12, 10, 16, seed=5, diagonal_boost=1e-2)
    shards, _ = local_solver(spec, 4, P.Backend.GRAPH_COLORED)
    assert all(_mesh_fused(s) for s in shards)
    rep_f, xs_f = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    monkeypatch.setenv("B2S_FUSE", "0")
    rep_u, xs_u = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    xf = np.concatenate([v.cpu().numpy() for v in xs_f])
    xu = np.concatenate([v.cpu().numpy() for v in xs_u])
    assert rep_f.converged and rep_u.converged
    assert abs(rep_f.iterations - rep_u.iterations) <= max(1.0, 0.1 * rep_u.iterations)
    assert np.linalg.norm(xf - xu) <= 1e-7 * np.linalg.norm(xu)


@pytest.mark.parametrize("backend", ["level", "color"])
def test_mesh_budget_exhaustion_reports_true_residual(backend):
    """Non-converged sharded solve: the final true residual needs x's ghost
    rows and an all-reduce (k_mesh_scalar) -- every shard reports the same
    global norm, equal to the host loop's."""
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    spec = P.GeneratorSpec(10, 8, 12, seed=5, diagonal_boost=1e-4)
    shards, comm = local_solver(spec, 3, P.Backend.from_name(backend))
    stop = P.StoppingCriteria(1e-12, 3)
    rep, xs = solve_shards_mesh(shards, stop)
    rep_h, xs_h = solve_shards(shards, comm, stop)
    assert not rep.converged and rep.failure_reason == "budget" and rep.iterations == 3.0
    assert rep_h.iterations == 3.0
    np.testing.assert_allclose(rep.final_norm, rep_h.final_norm, rtol=1e-8)
    x = np.concatenate([v.cpu().numpy() for v in xs])
    xh = np.concatenate([v.cpu().numpy() for v in xs_h])
    assert np.linalg.norm(x - xh) <= 1e-8 * np.linalg.norm(xh)


def test_mesh_halo_overlap_branch(monkeypatch):
    """B2S_MESH_OVERLAP=1: the halo runs on a side branch of the iteration
    graph, concurrent with the colour-1 SpMV -- same bits as in line."""
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    spec = P.GeneratorSpec(12, 10, 16, seed=5, diagonal_boost=1e-2)
    shards, _ = local_solver(spec, 4, P.Backend.GRAPH_COLORED)
    monkeypatch.setenv("B2S_MESH_OVERLAP", "0")
    rep0, xs0 = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    monkeypatch.setenv("B2S_MESH_OVERLAP", "1")
    rep1, xs1 = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    assert rep0.iterations == rep1.iterations
    for a, b in zip(xs0, xs1):
        assert torch.equal(a, b)


@pytest.mark.parametrize("backend", ["level", "color"])
def test_mesh_nonzero_initial_guess(backend):
    """x0 != 0: the initial residual takes x0's ghost rows (and, for fused
    2-colour shards, the local block plus the residual-mode ghost correction)."""
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    spec = P.GeneratorSpec(10, 8, 12, seed=5, diagonal_boost=1e-2)
    shards, comm = local_solver(spec, 3, P.Backend.from_name(backend))
    rng = np.random.default_rng(11)
    x0 = [rng.uniform(-1, 1, s.R * s.b) for s in shards]
    stop = P.StoppingCriteria(1e-8, 200)
    rep, xs = solve_shards_mesh(shards, stop, x0=x0)
    rep_h, xs_h = solve_shards(shards, comm, stop, x0=x0)
    assert rep.converged and rep_h.converged
    np.testing.assert_allclose(rep.initial_norm, rep_h.initial_norm, rtol=1e-12)
    assert abs(rep.iterations - rep_h.iterations) <= max(1.0, 0.1 * rep_h.iterations)
    x = np.concatenate([v.cpu().numpy() for v in xs])
    xh = np.concatenate([v.cpu().numpy() for v in xs_h])
    assert np.linalg.norm(x - xh) <= 1e-6 * np.linalg.norm(xh)


@pytest.mark.parametrize("backend", ["level", "color"])
def test_sharded_host_loop_matches_partitioned_oracle_per_plan(backend):
    """Colour shards too (not only level): the host-driven sharded loop
    against the reference's partitioned recipe with the same plan."""
    spec = P.GeneratorSpec(8, 7, 12, seed=5, diagonal_boost=1e-2)
    tol = 1e-8
    xo, ro = oracle_partitioned(spec, 2, tol, backend)
    shards, comm = local_solver(spec, 2, P.Backend.from_name(backend))
    rep, xs = solve_shards(shards, comm, P.StoppingCriteria(tol, 200))
    x = np.concatenate([v.cpu().numpy() for v in xs])
    assert rep.converged and ro.converged
    assert abs(rep.iterations - ro.iterations) <= max(1.0, 0.1 * ro.iterations)
    assert np.linalg.norm(x - xo) <= 1e-6 * np.linalg.norm(xo)


def test_mesh_dead_peer_times_out_instead_of_hanging(monkeypatch):
    """A shard whose peer never runs: its bounded device waits expire, the
    abort word goes up on every rank and the solve raises PeerTimeout
    (B2S_PEER_TIMEOUT) within the configured timeout instead of spinning
    forever (csrc/ctl.cuh wait_ge)."""
    import time

    from paper_2309_11488_b200._lib import PeerTimeout
    from paper_2309_11488_b200.distributed import (_mesh_krylov, _mesh_prepare, _mesh_struct)
    monkeypatch.setenv("B2S_MESH_TIMEOUT_MS", "300")
    spec = P.GeneratorSpec(8, 7, 12, seed=5, diagonal_boost=1e-2)
    shards, _ = local_solver(spec, 2, P.Backend.LEVEL_SCHEDULED)
    mss = [_mesh_prepare(s, 2) for s in shards]
    ptrs = [s.mesh.local_ptrs() for s in shards]
    s = shards[0]
    mss[0].peers = ptrs
    owner_rows = {h: shards[h].send[0].cpu().numpy() for h in s.recv}
    mesh, keep = _mesh_struct(s, mss[0], owner_rows, shared_device=True)
    kr = _mesh_krylov(s, mss[0])
    t0 = time.perf_counter()
    with pytest.raises(PeerTimeout):
        kr.solve(s.rhs_p, mss[0].x, P.StoppingCriteria(1e-8, 200), mesh=mesh, x0_zero=True)
    assert time.perf_counter() - t0 < 60.0
    # the abort word is up on the silent peer too
    assert int(shards[1].mesh.mbox[-8:].view(torch.int64)[0].item()) == 1
    torch.cuda.synchronize()
    # after a PeerTimeout the mesh state is rebuilt (sequence numbers and
    # abort words start afresh) and the shards solve normally
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    monkeypatch.delenv("B2S_MESH_TIMEOUT_MS")
    for sh in shards:
        sh.mesh = None
    rep, _ = solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))
    assert rep.converged


def test_mesh_needs_enough_hardware_queues(monkeypatch):
    from paper_2309_11488_b200.distributed import solve_shards_mesh
    spec = P.GeneratorSpec(8, 7, 12, seed=5, diagonal_boost=1e-2)
    shards, _ = local_solver(spec, 4, P.Backend.LEVEL_SCHEDULED)
    monkeypatch.setenv("CUDA_DEVICE_MAX_CONNECTIONS", "4")
    with pytest.raises(RuntimeError, match="CUDA_DEVICE_MAX_CONNECTIONS"):
        solve_shards_mesh(shards, P.StoppingCriteria(1e-8, 200))


def _torchrun(args, world, timeout=300):
    import socket
    import subprocess
    import sys
    from pathlib import Path
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    root = Path(__file__).resolve().parents[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1", f"--master-port={port}",
           *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=root)


def test_nccl_comm_host_loop_two_processes():
    """NcclComm (the host-driven sharded loop over torch.distributed) in two
    processes on the one GPU: NCCL refuses two ranks on one device, so the
    group is gloo here (halos and partial sums staged through the host);
    the same code path runs over NCCL on one GPU per rank."""
    import json
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = _torchrun([str(root / "tests" / "workers" / "mesh_worker.py"), "8,7,12", "color",
                     "--same-gpu", "--comm-loop"], 2)
    assert out.returncode == 0, out.stderr[-3000:]
    got = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    spec = P.GeneratorSpec(8, 7, 12, seed=5, diagonal_boost=1e-2)
    shards, comm = local_solver(spec, 2, P.Backend.GRAPH_COLORED)
    rep, xs = solve_shards(shards, comm, P.StoppingCriteria(1e-8, 200))
    x = np.concatenate([v.cpu().numpy() for v in xs])
    assert all(got["converged"])
    assert got["iterations"][0] == rep.iterations
    assert np.linalg.norm(np.asarray(got["x"]) - x) <= 1e-12 * np.linalg.norm(x)


def test_mesh_unavailable_is_agreed_and_falls_back():
    """One rank cannot open its peers' IPC buffers: every rank raises
    MeshUnavailable at the same point (no rank is left waiting on a peer)
    and the solve completes on the host-driven loop instead."""
    import json
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = _torchrun([str(root / "tests" / "workers" / "mesh_worker.py"), "8,7,12", "color",
                     "--same-gpu", "--fail-ipc-rank", "1"], 2)
    assert out.returncode == 0, out.stderr[-3000:]
    got = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert got["fallback"] and "rank 1" in got["fallback"]
    assert all(got["converged"]) and got["rerun_bit_equal"]


def test_nccl_comm_world_of_one_over_nccl():
    """The same host loop over a real NCCL communicator (one rank)."""
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = _torchrun([str(root / "bench.py"), "--gpus", "1", "--force-dist", "--dist-comm", "nccl",
                     "--grid", "24,20,16", "--steps", "2", "--warmup", "1", "--no-e2e",
                     "--no-cpu"], 1)
    assert out.returncode == 0, out.stderr[-3000:]
    import json
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["value"] > 0 and line.get("converged", True)


def test_device_halo_plan_equals_host_halo_plan():
    """The shard derives its halo bookkeeping on the device from the uploaded
    slab; it must equal the host HaloPlan (ghost ids, owners, local columns,
    the diagonal block's pattern)."""
    from paper_2309_11488_b200.distributed import HaloPlan, Shard, generate_slab
    spec = P.GeneratorSpec(9, 7, 12, seed=5)
    world = 3
    owners = np.array([slab_bounds(spec.nz, world, r)[0] * spec.nx * spec.ny
                       for r in range(world)], dtype=np.int64)
    for r in range(world):
        slab = generate_slab(spec, r, world)
        hp = HaloPlan(slab, owners)
        sh = Shard(slab, owners, None)
        np.testing.assert_array_equal(sh.ghosts, hp.ghosts)
        assert sorted(sh.recv) == sorted(hp.recv)
        for h in hp.recv:
            np.testing.assert_array_equal(sh.recv[h], hp.recv[h])
        np.testing.assert_array_equal(sh.obsr.pat.ci[: sh.obsr.pat.nnz].cpu().numpy(), hp.lcol)
        rows = np.repeat(np.arange(slab.rows), np.diff(slab.rp))
        prp = np.zeros(slab.rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows[hp.own], minlength=slab.rows), out=prp[1:])
        pat = sh.pmat.pattern
        np.testing.assert_array_equal(pat.row_pointers, prp)
        np.testing.assert_array_equal(pat.column_indices, hp.lcol[hp.own])
