"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container only (the reference does not exist on the GPU
box):  python tests/golden/make_golden.py
It imports ``blocksolve`` from /root/reference/pkg/src (read-only; byte-code
writing disabled), runs the reference's own functions on seeded inputs and
stores inputs + outputs as compressed .npz files next to this script.  The
oracle port (oracle/port.py) and the CUDA path are both checked against
these files by tests/.
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

import blocksolve as bs  # noqa: E402
from blocksolve.io import GeneratorSpec, generate  # noqa: E402
from blocksolve.krylov import dot_partials, norm_array  # noqa: E402

OUT = Path(__file__).resolve().parent
RNG = np.random.default_rng(20240817)


def pattern_from_rows(rows, n):
    rp = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for r in range(n):
        cs = sorted(set(rows.get(r, [])))
        rp[r + 1] = rp[r] + len(cs)
        cols.extend(cs)
    return bs.SparsityPattern(n, rp, np.array(cols, dtype=np.int64))


def dominant(p, b, rng):
    nnz = p.num_blocks
    vals = rng.uniform(-1.0, 1.0, size=(nnz, b, b))
    rows = np.repeat(np.arange(p.num_block_rows), np.diff(p.row_pointers))
    off = rows != p.column_indices
    sums = np.zeros((p.num_block_rows, b))
    np.add.at(sums, rows[off], np.abs(vals[off]).sum(axis=2))
    d = np.flatnonzero(~off)
    vals[d] = 0.0
    vals[d[:, None], np.arange(b)[None, :], np.arange(b)[None, :]] = sums[rows[d]] + 1.0
    return vals.reshape(-1)


def plan_dict(prefix, plan):
    return {f"{prefix}_row_group": plan.row_group, f"{prefix}_perm": plan.permutation,
            f"{prefix}_iperm": plan.inverse_permutation, f"{prefix}_offsets": plan.group_offsets}


def system_case(name, a, rhs, strategies=("level", "color", "sequential"), tols=(0.01, 1e-8)):
    out = {"rp": a.pattern.row_pointers, "ci": a.pattern.column_indices,
           "vals": a.values, "b": np.array(a.block_size), "rhs": rhs.data}
    p = a.pattern
    plans = {"level": bs.level_schedule(p), "color": bs.graph_color(p),
             "sequential": bs.sequential_plan(p.num_block_rows)}
    x = RNG.uniform(-1, 1, size=rhs.data.size)
    out["x"] = x
    out["spmv"] = bs.spmv(a, bs.BlockVector(x, a.block_size)).data
    out["dot_xx"] = np.array(bs.dot(bs.BlockVector(x, a.block_size),
                                    bs.BlockVector(x, a.block_size)))
    for s in strategies:
        plan = plans[s]
        out.update(plan_dict(s, plan))
        f = bs.decompose(a, plan)
        out[f"{s}_lu_perm_rp"] = f.combined.pattern.row_pointers
        out[f"{s}_lu_perm_ci"] = f.combined.pattern.column_indices
        out[f"{s}_lu"] = f.combined.values
        out[f"{s}_invd"] = f.inverted_diagonals.reshape(-1)
        out[f"{s}_apply"] = f.apply(bs.BlockVector(x, a.block_size)).data
        for tol in tols:
            xs, rep = bs.bicgstab(bs.MatrixOperator(a), f, rhs,
                                  stop=bs.StoppingCriteria(tol, 200))
            tag = f"{s}_tol{tol:g}"
            out[f"{tag}_x"] = xs.data
            out[f"{tag}_report"] = np.array([rep.converged, rep.iterations, rep.initial_norm,
                                             rep.final_norm], dtype=np.float64)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(name, {k: v.shape for k, v in out.items() if v.size > 1000})


def main():
    # C1: the BASELINE config-0 system (20x20x10, seed 0), full pipeline
    c1 = generate(GeneratorSpec(20, 20, 10, seed=0))
    system_case("c1_20x20x10", c1.a, c1.rhs)
    # a small generator case with non-default recipe (tz, boost), b = 2
    s2 = generate(GeneratorSpec(6, 5, 4, block_size=2, tz=0.1, diagonal_boost=0.05, seed=31))
    system_case("gen_6x5x4_b2", s2.a, s2.rhs)
    # b = 1 generator case
    s1 = generate(GeneratorSpec(7, 3, 5, block_size=1, seed=5))
    system_case("gen_7x3x5_b1", s1.a, s1.rhs)

    # random non-symmetric patterns (analysis + factor + apply), b = 3
    pats = {}
    for t in range(12):
        n = int(RNG.integers(5, 60))
        rows = {i: {i} for i in range(n)}
        for _ in range(int(RNG.integers(n, 4 * n))):
            i, j = (int(v) for v in RNG.integers(0, n, size=2))
            rows[i].add(j)
        p = pattern_from_rows({r: list(c) for r, c in rows.items()}, n)
        b = int(RNG.integers(1, 4))
        a = bs.BlockMatrix(p, b, dominant(p, b, RNG))
        rhs = bs.BlockVector(RNG.uniform(-1, 1, size=n * b), b)
        lev, col = bs.level_schedule(p), bs.graph_color(p)
        x = RNG.uniform(-1, 1, size=n * b)
        entry = {"rp": p.row_pointers, "ci": p.column_indices, "vals": a.values,
                 "b": np.array(b), "x": x, "rhs": rhs.data,
                 "spmv": bs.spmv(a, bs.BlockVector(x, b)).data}
        entry.update(plan_dict("level", lev))
        entry.update(plan_dict("color", col))
        for s, plan in (("level", lev), ("color", col)):
            f = bs.decompose(a, plan)
            entry[f"{s}_lu"] = f.combined.values
            entry[f"{s}_lu_perm_ci"] = f.combined.pattern.column_indices
            entry[f"{s}_invd"] = f.inverted_diagonals.reshape(-1)
            entry[f"{s}_apply"] = f.apply(bs.BlockVector(x, b)).data
            entry[f"{s}_inorder"] = f.factors_in_input_order().values
        for k, v in entry.items():
            pats[f"r{t}_{k}"] = v
    np.savez_compressed(OUT / "random_patterns.npz", **pats)

    # hand cases: scalar 2x2 (bs tests: [4,2,0.25,2.5]), chain, clique, partials
    hand = {}
    m = bs.BlockMatrix.from_blocks([(0, 0, np.array([[4.0]])), (0, 1, np.array([[2.0]])),
                                    (1, 0, np.array([[1.0]])), (1, 1, np.array([[3.0]]))])
    hand["scalar_lu"] = bs.decompose(m, bs.sequential_plan(2)).combined.values
    chain = pattern_from_rows({0: [0], 1: [0, 1], 2: [1, 2]}, 3)
    hand["chain_levels"] = bs.level_schedule(chain).row_group
    hand["chain_colors"] = bs.graph_color(chain).row_group
    clique = pattern_from_rows({i: list(range(4)) for i in range(4)}, 4)
    hand["clique_colors"] = bs.graph_color(clique).row_group
    hand["partials_130"] = dot_partials(np.ones(130), np.ones(130))
    v = RNG.standard_normal(4099)
    hand["dot_v"] = v
    hand["dot_vv"] = np.array(bs.dot(bs.BlockVector(v, 1), bs.BlockVector(v, 1)))
    hand["norm_v"] = np.array(norm_array(v))
    # Block-Jacobi: 12x12x8 stencil, two z-slabs
    g = generate(GeneratorSpec(12, 12, 8, seed=3))
    part = (np.arange(g.a.num_block_rows) // (12 * 12 * 4)).astype(np.int64)
    jac, cp = bs.drop_cross_blocks(g.a, bs.Partitioning(2, part, 0.0))
    hand["jac_rp"] = jac.pattern.row_pointers
    hand["jac_ci"] = jac.pattern.column_indices
    hand["jac_idx"] = cp.indices
    hand["jac_part"] = part
    f = bs.decompose(jac, bs.level_schedule(jac.pattern))
    xs, rep = bs.bicgstab(bs.MatrixOperator(g.a), f, g.rhs, stop=bs.StoppingCriteria(1e-8, 200))
    hand["jac_report"] = np.array([rep.converged, rep.iterations, rep.initial_norm,
                                   rep.final_norm])
    hand["jac_x"] = xs.data
    # generator digests for larger grids (bit-exact generator check)
    for dims in ((20, 20, 10), (30, 17, 9)):
        gg = generate(GeneratorSpec(*dims, seed=0))
        hand[f"gen_{'x'.join(map(str, dims))}_sum"] = np.array(
            [gg.a.values.sum(), np.abs(gg.a.values).sum(), gg.rhs.data.sum(),
             float(gg.a.pattern.column_indices.sum())])
    np.savez_compressed(OUT / "hand_cases.npz", **hand)


if __name__ == "__main__":
    main()
