"""Wells against the reference-generated
fixtures (tests/golden/make_wells.py): the generator's wells draw for draw,
coupled folding on the host (CPU), separately applied well terms on the
device and full solves in both well modes (GPU)."""

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

import paper_2309_11488_b200 as P

CASES = {
    "wells_std_8x7x5": dict(nx=8, ny=7, nz=5, well_count=3, well_kind="standard", seed=4),
    "wells_ms_8x7x5": dict(nx=8, ny=7, nz=5, well_count=2, well_kind="multisegment", seed=5),
    "wells_std_b2_6x6x4": dict(nx=6, ny=6, nz=4, block_size=2, well_count=2,
                               well_kind="standard", well_depth=4, seed=6),
}


def close(got, ref, rel):
    scale = max(np.abs(ref).max(), 1e-300)
    assert_allclose(got, ref, rtol=0, atol=rel * scale)


@pytest.mark.parametrize("name", CASES)
def test_generator_wells_draw_for_draw(golden, name):
    g, ref = P.generate(P.GeneratorSpec(**CASES[name])), golden(name)
    assert_array_equal(g.a.values, ref["vals"])
    assert_array_equal(g.rhs.data, ref["rhs"])
    for k, w in enumerate(g.wells.standard):
        assert_array_equal(w.perforated_cells, ref[f"std{k}_cells"])
        assert_array_equal(w.b_blocks, ref[f"std{k}_b"])
        assert_array_equal(w.c_blocks, ref[f"std{k}_c"])
        assert_array_equal(w.d_inverse, ref[f"std{k}_dinv"])
    for k, w in enumerate(g.wells.multisegment):
        assert_array_equal(w.b_cells, ref[f"ms{k}_cells"])
        assert_array_equal(w.b_blocks, ref[f"ms{k}_b"])
        assert_array_equal(w.d_dense, ref[f"ms{k}_d"])


@pytest.mark.parametrize("name", CASES)
def test_fold_into_matrix(golden, name):
    """Coupled mode folds C^T D^-1 B into A on the host (bs/wells.py:218-283)."""
    g, ref = P.generate(P.GeneratorSpec(**CASES[name])), golden(name)
    f = P.fold_into_matrix(g.a, g.wells)
    assert_array_equal(f.pattern.row_pointers, ref["fold_rp"])
    assert_array_equal(f.pattern.column_indices, ref["fold_ci"])
    close(f.values, ref["fold_vals"], 1e-14)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_well_augmented_operator_on_device(golden, name):
    g, ref = P.generate(P.GeneratorSpec(**CASES[name])), golden(name)
    op = P.WellAugmentedOperator(g.a, g.wells)
    close(op.apply_array(ref["x"]), ref["op_x"], 1e-13)
    # the public per-well entry points agree with the set
    y = P.spmv(g.a, P.BlockVector(ref["x"], g.a.block_size))
    for w in g.wells.standard:
        P.apply_standard(w, P.BlockVector(ref["x"], g.a.block_size), y)
    for w in g.wells.multisegment:
        P.apply_multisegment(w, P.BlockVector(ref["x"], g.a.block_size), y)
    close(y.data, ref["op_x"], 1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("mode", ["separate", "coupled"])
@pytest.mark.parametrize("backend", ["level", "color"])
def test_solve_with_wells(golden, name, mode, backend):
    g, ref = P.generate(P.GeneratorSpec(**CASES[name])), golden(name)
    cfg = P.SolverConfig(backend=P.Backend.from_name(backend), well_mode=P.WellMode(mode),
                         stop=P.StoppingCriteria(1e-8, 200))
    x, rep = P.solve_with_fallback(cfg, g.a, g.rhs, g.wells)
    conv, its, n0, fin, fb = ref[f"{mode}_{backend}_report"]
    assert rep.converged and not rep.fallback_used
    assert abs(rep.iterations - its) <= 1.0, (rep.iterations, its)
    assert_allclose(rep.initial_norm, n0, rtol=1e-12)
    xr = ref[f"{mode}_{backend}_x"]
    assert np.linalg.norm(x.data - xr) <= 1e-7 * np.linalg.norm(xr)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("backend", ["level", "color"])
def test_wells_in_device_loop_match_host_loop(name, backend):
    """Separate wells run inside the device-resident CUDA-graph loop (their
    terms subtracted in the SpMV epilogue, csrc/wells.cu + csrc/spmv.cu):
    same iterations and solution as the host-driven loop applying the
    same well kernels after each SpMV."""
    from paper_2309_11488_b200.krylov import _bicgstab_generic
    g = P.generate(P.GeneratorSpec(**CASES[name]))
    plan = (P.level_schedule if backend == "level" else P.graph_color)(g.a.pattern)
    fact = P.decompose(g.a, plan)
    op = P.WellAugmentedOperator(g.a, g.wells)
    stop = P.StoppingCriteria(1e-8, 200)
    x_dev, r_dev = P.bicgstab(op, fact, g.rhs, stop=stop)
    assert r_dev.gpu_launches > 0          # the native graph loop ran
    x0 = P.BlockVector.zeros(g.a.num_block_rows, g.a.block_size)
    x_host, r_host = _bicgstab_generic(op, fact, g.rhs, x0, stop)
    assert r_dev.converged and r_host.converged
    assert abs(r_dev.iterations - r_host.iterations) <= 0.5
    assert r_dev.initial_norm == r_host.initial_norm
    assert np.linalg.norm(x_dev.data - x_host.data) <= 1e-9 * np.linalg.norm(x_host.data)
    # and through the bridge, with an initial guess
    x0 = P.BlockVector(np.full(g.rhs.data.size, 0.05), g.a.block_size)
    cfg = P.SolverConfig(backend=P.Backend.from_name(backend), stop=stop)
    x_b, r_b = P.solve_with_fallback(cfg, g.a, g.rhs, g.wells, x0=x0)
    from paper_2309_11488_b200.krylov import norm_array
    assert r_b.converged and r_b.gpu_launches > 0
    assert r_b.initial_norm == norm_array(g.rhs.data - op.apply_array(x0.data))


@pytest.mark.gpu
@pytest.mark.parametrize("vec,simg", [("1", "1"), ("0", "1"), ("0", "0")])
def test_wells_with_fused_colour_passes(monkeypatch, vec, simg):
    """2-colour plans keep the fused colour passes with separate wells: the
    colour-0 rows of v / t get their well terms after p^ / s^ is complete
    (k_wells_patch, partials corrected; under the s-image it also recomputes
    u = inv(A_ii) v at the patched rows and the colour-1 SpMV subtracts the
    terms before forming F(v)); same answer as the unfused loop."""
    from paper_2309_11488_b200.krylov import DeviceKrylov
    monkeypatch.setenv("B2S_FUSE_VEC", vec)
    monkeypatch.setenv("B2S_SIMG", simg)
    g = P.generate(P.GeneratorSpec(14, 12, 10, well_count=4, well_depth=6, seed=21))
    fact = P.decompose(g.a, P.graph_color(g.a.pattern))
    op = P.WellAugmentedOperator(g.a, g.wells)
    stop = P.StoppingCriteria(1e-10, 200)
    assert DeviceKrylov.build(g.a, fact, wells=g.wells).fuse
    x_f, r_f = P.bicgstab(op, fact, g.rhs, stop=stop)
    monkeypatch.setenv("B2S_FUSE", "0")
    assert not DeviceKrylov.build(g.a, fact, wells=g.wells).fuse
    x_u, r_u = P.bicgstab(op, fact, g.rhs, stop=stop)
    assert r_f.converged and r_u.converged
    assert abs(r_f.iterations - r_u.iterations) <= 0.5
    assert np.linalg.norm(x_f.data - x_u.data) <= 1e-9 * np.linalg.norm(x_u.data)
    y = op.apply_array(x_f.data)
    assert np.linalg.norm(g.rhs.data - y) <= 1e-10 * np.linalg.norm(g.rhs.data) * 1.01
