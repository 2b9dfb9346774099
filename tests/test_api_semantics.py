"""API semantics the reference has and a device port could lose: bundle
signature and shape checks (bs/io.py:33-44), COUPLED well sets add nothing
in the operator (bs/krylov.py:84-94 via bs/wells.py:187-202), and in-place
changes of host arrays between calls are seen (the reference reads the host
arrays at every apply)."""

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

import paper_2309_11488_b200 as P


def test_system_bundle_reference_signature():
    g = P.generate(P.GeneratorSpec(3, 3, 2, well_count=1, well_depth=2, seed=1))
    b = P.SystemBundle(g.a, g.rhs, g.wells, P.BundleMeta("x", 3, (3, 3, 2)))
    assert b.wells is g.wells and b.meta.name == "x"
    assert g.meta == P.BundleMeta("synthetic-3x3x2", 3, (3, 3, 2))
    with pytest.raises(P.ShapeError):
        P.SystemBundle(g.a, P.BlockVector(np.zeros(9), 3), g.wells, g.meta)
    with pytest.raises(P.ShapeError):
        P.SystemBundle(g.a, P.BlockVector(np.zeros(g.rhs.data.size), 1), g.wells, g.meta)


def test_bundle_round_trip_keeps_wells(tmp_path):
    g = P.generate(P.GeneratorSpec(4, 3, 3, well_count=2, well_depth=2, seed=2))
    P.write_system(g, tmp_path / "case.mtx")
    back = P.read_system(tmp_path / "case.mtx")
    assert back.meta.name == "case" and len(back.wells.standard) == 2
    assert_array_equal(back.a.values, g.a.values)


@pytest.mark.gpu
def test_coupled_set_adds_nothing_in_the_operator():
    g = P.generate(P.GeneratorSpec(5, 4, 4, well_count=2, well_depth=3, seed=3))
    coupled = P.WellSet(g.wells.standard, g.wells.multisegment, P.WellMode.COUPLED)
    x = np.random.default_rng(0).uniform(-1, 1, g.rhs.data.size)
    plain = P.MatrixOperator(g.a).apply_array(x)
    assert_array_equal(P.WellAugmentedOperator(g.a, coupled).apply_array(x), plain)
    assert_array_equal(P.WellAugmentedOperator(g.a, P.WellSet()).apply_array(x), plain)
    sep = P.WellAugmentedOperator(g.a, g.wells).apply_array(x)
    assert not np.array_equal(sep, plain)


@pytest.mark.gpu
def test_in_place_changes_are_seen_between_calls():
    g = P.generate(P.GeneratorSpec(5, 4, 4, well_count=1, well_depth=3,
                                   well_kind="multisegment", seed=4))
    x = np.random.default_rng(1).uniform(-1, 1, g.rhs.data.size)
    op = P.WellAugmentedOperator(g.a, g.wells)
    y0 = op.apply_array(x)
    # matrix values changed in place
    g.a.values *= 2.0
    y1 = op.apply_array(x)
    assert not np.array_equal(y0, y1)
    # a well's D changed in place and refactored (bs/wells.py:106-114)
    w = g.wells.multisegment[0]
    w.d_dense *= 3.0
    w._refactor()
    y2 = op.apply_array(x)
    want = P.spmv(g.a, P.BlockVector(x, 3)).data.copy()
    g.wells.apply_contributions_array(x, want, 3)
    assert not np.array_equal(y1, y2)
    assert_allclose(y2, want, rtol=0, atol=1e-13 * np.abs(want).max())
    # a well appended
    extra = P.generate(P.GeneratorSpec(5, 4, 4, well_count=1, well_depth=2, seed=9)).wells
    g.wells.standard.extend(extra.standard)
    y3 = op.apply_array(x)
    assert not np.array_equal(y2, y3)


@pytest.mark.gpu
def test_bicgstab_operator_reads_current_values():
    """decompose(A) then A.values changed: the operator uses the new values,
    the preconditioner the old ones -- as in the reference."""
    g = P.generate(P.GeneratorSpec(6, 5, 4, seed=5))
    for plan in (P.graph_color, P.level_schedule):
        a = P.BlockMatrix(g.a.pattern, 3, g.a.values.copy())
        fact = P.decompose(a, plan(a.pattern))
        a.values *= 1.5
        x, rep = P.bicgstab(P.MatrixOperator(a), fact, g.rhs,
                            stop=P.StoppingCriteria(1e-10, 200))
        assert rep.converged
        r = g.rhs.data - P.spmv(a, x).data
        assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(g.rhs.data) * 1.01


@pytest.mark.gpu
def test_staged_pageable_upload_is_exact():
    """Pageable host arrays reach the device through the page-locked staging
    ring (paper_2309_11488_b200/_device.py staged_copy) byte for byte, for
    sizes around the chunk size, and a pageable solve equals a pinned one."""
    import torch

    from paper_2309_11488_b200 import _device as D
    rng = np.random.default_rng(4)
    C = D.STAGE_CHUNK // 8
    # (arrays of a few chunks are cut into >= 1 MB pieces: both regimes)
    for n in (1, 1000, (1 << 17) - 1, (1 << 17) + 3, C - 1, C, C + 1, 3 * C + 17, 9 * C + 5):
        a = rng.standard_normal(n)
        d = D.to_device(torch.from_numpy(a), torch.device("cuda"))
        torch.cuda.synchronize()
        assert_array_equal(d.cpu().numpy(), a)
    # int64 indices narrowed to int32 while staging
    for n in (1, 5000, (C * 2) + 7, 3 * C + 1):
        a = rng.integers(0, 2**31 - 1, size=n, dtype=np.int64)
        d = torch.empty(n, dtype=torch.int32, device="cuda")
        D.staged_copy(d, torch.from_numpy(a), torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert_array_equal(d.cpu().numpy(), a.astype(np.int32))
    g = P.generate(P.GeneratorSpec(60, 50, 40, seed=2))
    cfg = P.SolverConfig(backend=P.Backend.GRAPH_COLORED, stop=P.StoppingCriteria(1e-8, 200))
    x1, r1 = P.solve_with_fallback(cfg, g.a, g.rhs)
    x2, r2 = P.solve_with_fallback(cfg, P.pin_host(g.a), P.pin_host(g.rhs))
    assert_array_equal(x1.data, x2.data)
    assert r1.iterations == r2.iterations


@pytest.mark.gpu
def test_concurrent_solves_from_threads_match_sequential():
    """Independent systems solved concurrently from several host threads (the
    reference CLI's --parallel pool; SURVEY 8(b) "threading") give exactly
    the results of one-at-a-time solves: no shared mutable state on the
    solve path beyond thread-safe pools."""
    import concurrent.futures as cf
    cases = []
    for k, (dims, backend) in enumerate([((14, 12, 9), P.Backend.GRAPH_COLORED),
                                         ((20, 18, 12), P.Backend.LEVEL_SCHEDULED),
                                         ((16, 16, 6), P.Backend.REFERENCE_SEQUENTIAL),
                                         ((30, 10, 8), P.Backend.GRAPH_COLORED)]):
        g = P.generate(P.GeneratorSpec(*dims, seed=20 + k, well_count=1, well_depth=2))
        cases.append((P.SolverConfig(backend=backend, stop=P.StoppingCriteria(1e-9, 300)),
                      g.a, g.rhs, g.wells))

    def run(case):
        cfg, a, b, w = case
        x, rep = P.solve_with_fallback(cfg, a, b, w)
        return x.data.copy(), rep.iterations
    seq = [run(c) for c in cases]
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        par = list(ex.map(run, cases * 3))
    for i, (x, its) in enumerate(par):
        assert_array_equal(x, seq[i % len(cases)][0])
        assert its == seq[i % len(cases)][1]


@pytest.mark.gpu
@pytest.mark.parametrize("backend", [P.Backend.GRAPH_COLORED, P.Backend.LEVEL_SCHEDULED,
                                     P.Backend.REFERENCE_SEQUENTIAL])
def test_solve_session_equals_solve_with_fallback(backend):
    """A SolveSession (pattern phase once, values per solve) returns exactly
    what solve_with_fallback returns for each system: several value sets on
    one pattern, with wells and an initial guess, a singular system (through
    the fallback) and a system on another pattern (delegated)."""
    g = P.generate(P.GeneratorSpec(20, 18, 12, seed=3, well_count=2, well_depth=3))
    cfg = P.SolverConfig(backend=backend, stop=P.StoppingCriteria(1e-9, 300))
    sess = P.SolveSession(cfg, g.a.pattern, 3)
    rng = np.random.default_rng(5)
    for k in range(3):
        vals = g.a.values * (1.0 + 0.05 * rng.standard_normal(g.a.values.size))
        a = P.BlockMatrix(g.a.pattern, 3, vals)
        b = P.BlockVector(rng.uniform(-1, 1, g.rhs.data.size), 3)
        x0 = None if k == 0 else P.BlockVector(rng.uniform(-1, 1, b.data.size) * 1e-3, 3)
        w = g.wells if k == 2 else None
        x1, r1 = sess.solve(a, b, w, x0)
        x2, r2 = P.solve_with_fallback(cfg, a, b, w, x0)
        assert_array_equal(x1.data, x2.data)
        assert (r1.iterations, r1.converged, r1.fallback_used) == \
            (r2.iterations, r2.converged, r2.fallback_used)
        assert r1.initial_norm == r2.initial_norm and r1.final_norm == r2.final_norm
    # a pivot that is exactly zero at the corner row: both take the fallback path
    vals = g.a.values.copy()
    vals.reshape(-1, 3, 3)[g.a.pattern.position(0, 0)] = 0.0
    a = P.BlockMatrix(g.a.pattern, 3, vals)
    try:
        x2, r2 = P.solve_with_fallback(cfg, a, g.rhs)
        x1, r1 = sess.solve(a, g.rhs)
        assert_array_equal(x1.data, x2.data) and r1.fallback_used == r2.fallback_used
    except P.SolveFailed:
        with pytest.raises(P.SolveFailed):
            sess.solve(a, g.rhs)
    # another pattern: delegated
    h = P.generate(P.GeneratorSpec(8, 7, 6, seed=4))
    x1, r1 = sess.solve(h.a, h.rhs)
    x2, r2 = P.solve_with_fallback(cfg, h.a, h.rhs)
    assert_array_equal(x1.data, x2.data)
    sess.close()
