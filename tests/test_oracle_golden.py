"""The oracle port (oracle/port.py) against the reference-generated golden
fixtures: pins the checker before the CUDA path is judged by it.  CPU only."""

import numpy as np
import pytest
from numpy.testing import assert_allclose, assert_array_equal

from oracle import port as O


def _sys(g):
    b = int(g["b"])
    rp, ci = g["rp"], g["ci"]
    return rp, ci, g["vals"].reshape(-1, b, b), b


SYSTEMS = ["c1_20x20x10", "gen_6x5x4_b2", "gen_7x3x5_b1", "masked_14x16x8", "hetero_10x12x6"]


@pytest.mark.parametrize("name", SYSTEMS)
def test_plans_bit_exact(golden, name):
    g = golden(name)
    rp, ci, _, _ = _sys(g)
    lev = O.plan_from_groups(O.level_groups(rp, ci))
    col = O.plan_from_groups(O.color_groups(rp, ci))
    for tag, plan in (("level", lev), ("color", col)):
        assert_array_equal(plan.row_group, g[f"{tag}_row_group"])
        assert_array_equal(plan.permutation, g[f"{tag}_perm"])
        assert_array_equal(plan.inverse_permutation, g[f"{tag}_iperm"])
        assert_array_equal(plan.group_offsets, g[f"{tag}_offsets"])


@pytest.mark.parametrize("name", SYSTEMS)
@pytest.mark.parametrize("strategy", ["level", "color", "sequential"])
def test_factor_apply_solve(golden, name, strategy):
    g = golden(name)
    if f"{strategy}_lu" not in g:
        pytest.skip("fixture built for level/colour only")
    rp, ci, v3, b = _sys(g)
    plan = {"level": lambda: O.plan_from_groups(O.level_groups(rp, ci)),
            "color": lambda: O.plan_from_groups(O.color_groups(rp, ci)),
            "sequential": lambda: O.sequential(len(rp) - 1)}[strategy]()
    f = O.ilu0(rp, ci, v3, plan)
    assert_array_equal(f.rp, g[f"{strategy}_lu_perm_rp"])
    assert_array_equal(f.ci, g[f"{strategy}_lu_perm_ci"])
    ref = g[f"{strategy}_lu"]
    assert_allclose(f.lu.reshape(-1), ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    ref = g[f"{strategy}_invd"]
    assert_allclose(f.inv_diag.reshape(-1), ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    z = O.ilu0_apply(f, g["x"])
    ref = g[f"{strategy}_apply"]
    assert np.linalg.norm(z - ref) <= 1e-12 * np.linalg.norm(ref)
    assert_allclose(O.spmv(rp, ci, v3, g["x"]), g["spmv"], rtol=1e-13, atol=1e-13)
    for tol in (0.01, 1e-8):
        x, rep = O.bicgstab(lambda v: O.spmv(rp, ci, v3, v), lambda r: O.ilu0_apply(f, r),
                            g["rhs"], tol=tol)
        conv, its, n0, fin = g[f"{strategy}_tol{tol:g}_report"]
        assert rep.converged == bool(conv)
        assert rep.iterations == its
        assert_allclose(rep.initial_norm, n0, rtol=1e-13)
        assert_allclose(rep.final_norm, fin, rtol=1e-6)
        ref = g[f"{strategy}_tol{tol:g}_x"]
        assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)


def test_random_patterns(golden):
    g = golden("random_patterns")
    for t in range(12):
        e = {k[len(f"r{t}_"):]: v for k, v in g.items() if k.startswith(f"r{t}_")}
        b = int(e["b"])
        rp, ci, v3 = e["rp"], e["ci"], e["vals"].reshape(-1, b, b)
        assert_allclose(O.spmv(rp, ci, v3, e["x"]), e["spmv"], rtol=1e-13, atol=1e-13)
        for tag, groups in (("level", O.level_groups(rp, ci)), ("color", O.color_groups(rp, ci))):
            assert_array_equal(groups, e[f"{tag}_row_group"])
            plan = O.plan_from_groups(groups)
            assert_array_equal(plan.inverse_permutation, e[f"{tag}_iperm"])
            f = O.ilu0(rp, ci, v3, plan)
            assert_array_equal(f.ci, e[f"{tag}_lu_perm_ci"])
            assert_allclose(f.lu.reshape(-1), e[f"{tag}_lu"], atol=1e-12 * np.abs(e[f"{tag}_lu"]).max())
            _, _, back = O.factors_input_order(f)
            assert_allclose(back.reshape(-1), e[f"{tag}_inorder"],
                            atol=1e-12 * np.abs(e[f"{tag}_inorder"]).max())
            z = O.ilu0_apply(f, e["x"])
            assert np.linalg.norm(z - e[f"{tag}_apply"]) <= 1e-11 * np.linalg.norm(e[f"{tag}_apply"])


def test_hand_cases(golden):
    h = golden("hand_cases")
    rp = np.array([0, 2, 4]); ci = np.array([0, 1, 0, 1])
    v3 = np.array([4.0, 2.0, 1.0, 3.0]).reshape(4, 1, 1)
    f = O.ilu0(rp, ci, v3, O.sequential(2))
    assert_array_equal(f.lu.reshape(-1), h["scalar_lu"])
    assert_array_equal(h["scalar_lu"], [4.0, 2.0, 0.25, 2.5])
    chain_rp, chain_ci = np.array([0, 1, 3, 5]), np.array([0, 0, 1, 1, 2])
    assert_array_equal(O.level_groups(chain_rp, chain_ci), h["chain_levels"])
    assert_array_equal(O.color_groups(chain_rp, chain_ci), h["chain_colors"])
    assert_array_equal(O.dot_partials(np.ones(130), np.ones(130)), h["partials_130"])
    v = h["dot_v"]
    assert O.dot(v, v) == float(h["dot_vv"])


def test_jacobi_golden(golden):
    h = golden("hand_cases")
    from paper_2309_11488_b200.synthetic import GeneratorSpec, generate
    g = generate(GeneratorSpec(12, 12, 8, seed=3))
    a = g.a
    rp, ci = a.pattern.row_pointers, a.pattern.column_indices
    nrp, nci, nv, idx = O.drop_cross(rp, ci, a.values3d, h["jac_part"])
    assert_array_equal(nrp, h["jac_rp"])
    assert_array_equal(nci, h["jac_ci"])
    assert_array_equal(idx, h["jac_idx"])
    f = O.ilu0(nrp, nci, nv, O.plan_from_groups(O.level_groups(nrp, nci)))
    x, rep = O.bicgstab(lambda v: O.spmv(rp, ci, a.values3d, v), lambda r: O.ilu0_apply(f, r),
                        g.rhs.data, tol=1e-8)
    conv, its, n0, fin = h["jac_report"]
    assert rep.converged and rep.iterations == its


@pytest.mark.parametrize("name", ["c1_20x20x10", "gen_6x5x4_b2", "gen_7x3x5_b1"])
def test_generator_draw_for_draw(golden, name):
    """paper_2309_11488_b200.synthetic.generate == bs/io.py generate, bit for bit."""
    from paper_2309_11488_b200.synthetic import GeneratorSpec, generate
    spec = {"c1_20x20x10": GeneratorSpec(20, 20, 10, seed=0),
            "gen_6x5x4_b2": GeneratorSpec(6, 5, 4, block_size=2, tz=0.1, diagonal_boost=0.05, seed=31),
            "gen_7x3x5_b1": GeneratorSpec(7, 3, 5, block_size=1, seed=5)}[name]
    g = golden(name)
    s = generate(spec)
    assert_array_equal(s.a.pattern.row_pointers, g["rp"])
    assert_array_equal(s.a.pattern.column_indices, g["ci"])
    assert_array_equal(s.a.values, g["vals"])
    assert_array_equal(s.rhs.data, g["rhs"])


def test_generator_digests(golden):
    from paper_2309_11488_b200.synthetic import GeneratorSpec, generate
    h = golden("hand_cases")
    for dims in ((20, 20, 10), (30, 17, 9)):
        gg = generate(GeneratorSpec(*dims, seed=0))
        got = np.array([gg.a.values.sum(), np.abs(gg.a.values).sum(), gg.rhs.data.sum(),
                        float(gg.a.pattern.column_indices.sum())])
        assert_array_equal(got, h[f"gen_{'x'.join(map(str, dims))}_sum"])


@pytest.mark.parametrize("name,gen", [
    ("masked_14x16x8", lambda S: S.generate_masked(14, 16, 8, seed=11)),
    ("hetero_10x12x6", lambda S: S.generate_heterogeneous(10, 12, 6, sigma_k=1.5,
                                                          diagonal_boost=1e-3, seed=3))])
def test_config_generators_reproduce_fixtures(golden, name, gen):
    """The C2/C3 harness generators are seeded and deterministic: the
    fixtures the reference computed were built from exactly these arrays."""
    from paper_2309_11488_b200 import synthetic as S
    g, b = golden(name), gen(S)
    assert_array_equal(b.a.pattern.row_pointers, g["rp"])
    assert_array_equal(b.a.pattern.column_indices, g["ci"])
    assert_array_equal(b.a.values, g["vals"])
    assert_array_equal(b.rhs.data, g["rhs"])


def test_c2_masked_full_size_digest(golden):
    """C2 (46x112x22 masked, 47,605 cells): the oracle's plans equal the
    reference's bit for bit and its solves take the reference's iterations."""
    from paper_2309_11488_b200 import synthetic as S
    d = golden("c2_masked_digest")
    bnd = S.generate_masked(46, 112, 22, seed=2309)
    a = bnd.a
    rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
    assert a.num_block_rows == int(d["n"]) and a.pattern.num_blocks == int(d["nnzb"])
    lev, col = O.level_groups(rp, ci), O.color_groups(rp, ci)
    assert_array_equal(lev, d["level_row_group"])
    assert_array_equal(col, d["color_row_group"])
    f = O.ilu0(rp, ci, v3, O.plan_from_groups(col))
    x, rep = O.bicgstab(lambda v: O.spmv(rp, ci, v3, v), lambda r: O.ilu0_apply(f, r),
                        bnd.rhs.data, tol=1e-8)
    conv, its, n0, fin = d["color_report"]
    assert rep.converged and rep.iterations == its
    assert np.linalg.norm(x - d["color_x"]) <= 1e-8 * np.linalg.norm(d["color_x"])
