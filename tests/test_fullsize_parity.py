"""Full-size elementwise parity of the kernels that make the headline.

The BASELINE configs at their full sizes (C2 47,605 masked cells, C3
350,336 heterogeneous cells in two variants, C4 1,000,000 cells), both
parallel plans, through the public API:

* against the UNMODIFIED reference (tests/golden/make_fullsize.py ->
  full_<case>.npz): plan row_group / permutation sha256 (bit-exact), sampled
  plan-order L\\U blocks and inverse diagonals, SpMV and ILU0 apply of a
  seeded vector, and x after one BiCGStab iteration (the fused colour passes,
  the multi-slice SELL paths, factor2c and the phased two-entry sweeps all run
  at these sizes) -- elementwise within 1e-12 * max|ref|;
* against the oracle port run here on the same inputs: the COMPLETE factor,
  inverse-diagonal, SpMV and apply arrays (C2 and C4), same bar.

Errors are appended to $B2S_PARITY_LOG (JSON lines) when it is set.
"""

from __future__ import annotations

import hashlib
import json
import os
from pathlib import Path

import numpy as np
import pytest

import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import synthetic as S
from oracle import port as O

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = {
    "c2": lambda: S.generate_masked(46, 112, 22, seed=2309),
    "c3": lambda: S.generate_heterogeneous(92, 224, 17, sigma_k=1.0, diagonal_boost=1e-2),
    "c3s": lambda: S.generate_heterogeneous(92, 224, 17, sigma_k=2.0, diagonal_boost=1e-2),
    "c4": lambda: P.generate(P.GeneratorSpec(100, 100, 100, seed=0)),
}
PLANS = {"level": P.level_schedule, "color": P.graph_color}
TOL = 1e-12
_BUNDLES: dict = {}


def bundle(case):
    if case not in _BUNDLES:
        _BUNDLES.clear()            # one full-size system resident at a time
        _BUNDLES[case] = CASES[case]()
    return _BUNDLES[case]


def fixture(case, plan=None):
    p = GOLDEN / f"full_{case}_{plan}.npz"     # per-plan fixture with a solve band
    if plan is None or not p.exists():
        p = GOLDEN / f"full_{case}.npz"
    if not p.exists():
        pytest.skip(f"{p.name} not generated (tests/golden/make_fullsize.py {case})")
    with np.load(p) as z:
        return {k: z[k] for k in z.files}


def sha(a, dtype):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def log(**kw):
    path = os.environ.get("B2S_PARITY_LOG")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(kw) + "\n")


def rel_err(got, ref, scale):
    return float(np.abs(np.asarray(got) - np.asarray(ref)).max() / max(float(scale), 1e-300))


def check(name, got, ref, scale, bar=TOL, **ctx):
    e = rel_err(got, ref, scale)
    log(check=name, max_rel_err=e, bar=bar, **ctx)
    assert e <= bar, (name, e, ctx)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("plan", list(PLANS))
def test_fullsize_against_reference(case, plan):
    d = fixture(case, plan)
    bnd = bundle(case)
    a, rhs = bnd.a, bnd.rhs
    n, b = a.num_block_rows, a.block_size
    assert n == int(d["n"]) and a.pattern.num_blocks == int(d["nnzb"])
    blk, vec, rows = d["blk_idx"], d["vec_idx"], d["row_idx"]
    x = np.random.default_rng(99).uniform(-1.0, 1.0, n * b)   # make_fullsize.VEC_SEED

    y = P.spmv(a, P.BlockVector(x, b)).data
    check("spmv", y[vec], d["spmv_sample"], np.abs(y).max(), case=case)
    assert abs(np.linalg.norm(y) - float(d["spmv_norm"])) <= TOL * float(d["spmv_norm"])

    pl = PLANS[plan](a.pattern)
    assert pl.group_count == int(d[f"{plan}_groups"])
    assert sha(pl.row_group, np.int32) == str(d[f"{plan}_row_group_sha"])
    assert sha(pl.permutation, np.int64) == str(d[f"{plan}_perm_sha"])

    f = P.decompose(a, pl)
    lu = f.combined.values.reshape(-1, b, b)
    check("lu", lu[blk], d[f"{plan}_lu_sample"], d[f"{plan}_lu_absmax"], case=case, plan=plan)
    assert abs(np.linalg.norm(lu) / float(d[f"{plan}_lu_norm"]) - 1.0) <= TOL
    invd = f.inverted_diagonals.reshape(-1, b, b)
    check("invd", invd[rows], d[f"{plan}_invd_sample"], d[f"{plan}_invd_absmax"],
          case=case, plan=plan)
    assert abs(np.linalg.norm(invd) / float(d[f"{plan}_invd_norm"]) - 1.0) <= TOL
    z = f.apply(P.BlockVector(x, b)).data
    check("apply", z[vec], d[f"{plan}_apply_sample"], d[f"{plan}_apply_absmax"],
          case=case, plan=plan)

    # one BiCGStab iteration through the device loop (fused passes on 2 colours)
    x1, r1 = P.bicgstab(P.MatrixOperator(a), f, rhs, stop=P.StoppingCriteria(1e-8, 1))
    conv, its, n0, fin = d[f"{plan}_it1_report"]
    assert bool(r1.converged) == bool(conv) and r1.iterations == its
    assert r1.initial_norm == n0          # chunk-64 order, bit for bit
    check("bicgstab_1it_x", x1.data[vec], d[f"{plan}_it1_x_sample"], d[f"{plan}_it1_x_absmax"],
          case=case, plan=plan)
    assert abs(r1.final_norm - fin) <= 1e-10 * fin

    if f"{plan}_report" in d:   # the full solve, when the fixture has it
        conv, its, n0, fin = d[f"{plan}_report"]
        maxit = int(d.get(f"{plan}_maxit", 200))
        xs, rep = P.bicgstab(P.MatrixOperator(a), f, rhs, stop=P.StoppingCriteria(1e-8, maxit))
        assert rep.converged == bool(conv), (rep.converged, conv, rep.iterations, its)
        lo, hi = d[f"{plan}_band"] if f"{plan}_band" in d else (its, its)
        log(check="solve_iterations", case=case, plan=plan, gpu=rep.iterations, ref=float(its),
            band=[float(lo), float(hi)], converged=bool(rep.converged))
        assert lo - 1.0 <= rep.iterations <= hi + 1.0, (rep.iterations, its, lo, hi)
        assert rep.initial_norm == n0
        if not conv:   # both exhaust the budget (bs/krylov.py:242-244)
            assert rep.failure_reason == "budget" and rep.iterations == maxit
        elif case in ("c2", "c4"):   # well-conditioned: x itself agrees
            xr = d[f"{plan}_x_sample"]
            e = float(np.abs(xs.data[vec] - xr).max() / np.abs(xr).max())
            log(check="solve_x_sample", case=case, plan=plan, max_rel_err=e)
            assert e <= 1e-6
        else:   # ill-conditioned C3: the true residual meets the tolerance
            rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
            tr = np.linalg.norm(rhs.data - O.spmv(rp, ci, v3, xs.data))
            log(check="solve_true_residual", case=case, plan=plan, rel=tr / n0)
            assert tr <= 1e-8 * n0 * 1.01


@pytest.mark.slow
@pytest.mark.parametrize("case", ["c2", "c4"])
@pytest.mark.parametrize("plan", list(PLANS))
def test_fullsize_complete_arrays_against_oracle(case, plan):
    """Every element, not a sample: the oracle port (pinned to the reference
    bit for bit on the golden systems) run on the same full-size input."""
    bnd = bundle(case)
    a = bnd.a
    n, b = a.num_block_rows, a.block_size
    rp, ci, v3 = a.pattern.row_pointers, a.pattern.column_indices, a.values3d
    x = np.random.default_rng(99).uniform(-1.0, 1.0, n * b)
    yo = O.spmv(rp, ci, v3, x)
    check("spmv_full", P.spmv(a, P.BlockVector(x, b)).data, yo, np.abs(yo).max(),
          case=case, vs="oracle")
    groups = (O.level_groups if plan == "level" else O.color_groups)(rp, ci)
    plan_o = O.plan_from_groups(groups)
    fo = O.ilu0(rp, ci, v3, plan_o)
    pl = PLANS[plan](a.pattern)
    np.testing.assert_array_equal(pl.row_group, groups)
    f = P.decompose(a, pl)
    lu_o = fo.lu.reshape(-1)
    check("lu_full", f.combined.values, lu_o, np.abs(lu_o).max(), case=case, plan=plan,
          vs="oracle")
    invd_o = fo.inv_diag.reshape(-1)
    check("invd_full", f.inverted_diagonals.reshape(-1), invd_o, np.abs(invd_o).max(),
          case=case, plan=plan, vs="oracle")
    zo = O.ilu0_apply(fo, x)
    check("apply_full", f.apply(P.BlockVector(x, b)).data, zo, np.abs(zo).max(),
          case=case, plan=plan, vs="oracle")
