"""Golden partitions from the UNMODIFIED reference (bs/jacobi.py:46-108):
transmissibility_weights + partition on generator systems, masked and
heterogeneous harness systems and random non-symmetric patterns, for
several k.  Run in the build container only:
    python tests/golden/make_partitions.py
Writes tests/golden/partitions.npz.  Test infrastructure."""

from __future__ import annotations

import sys
from pathlib import Path

sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import blocksolve as bs  # noqa: E402

from paper_2309_11488_b200 import synthetic as S  # noqa: E402


def cases():
    yield "gen_6x5x4", bs.generate(bs.GeneratorSpec(6, 5, 4, seed=55)).a, (1, 6, 13)
    yield "gen_20x20x10", bs.generate(bs.GeneratorSpec(20, 20, 10, seed=77)).a, (150, 7)
    for name, b in (("masked_14x16x8", S.generate_masked(14, 16, 8, seed=11)),
                    ("hetero_10x12x6", S.generate_heterogeneous(10, 12, 6, sigma_k=1.5,
                                                                diagonal_boost=1e-3, seed=3))):
        a = b.a
        yield name, bs.BlockMatrix(bs.SparsityPattern(a.num_block_rows, a.pattern.row_pointers,
                                                      a.pattern.column_indices),
                                   a.block_size, a.values.copy()), (5, 33)
    rng = np.random.default_rng(4242)
    for t in range(6):
        n = int(rng.integers(8, 60))
        rows = {i: {i} for i in range(n)}
        for _ in range(int(rng.integers(n, 4 * n))):
            i, j = (int(v) for v in rng.integers(0, n, size=2))
            rows[i].add(j)
        rp = np.zeros(n + 1, dtype=np.int64)
        cols = []
        for r in range(n):
            cs = sorted(rows[r])
            rp[r + 1] = rp[r] + len(cs)
            cols += cs
        ci = np.array(cols, dtype=np.int64)
        vals = rng.uniform(-1, 1, size=ci.size * 4)
        yield f"random{t}", bs.BlockMatrix(bs.SparsityPattern(n, rp, ci), 2, vals), (2, n // 3)


def main():
    out = {}
    for name, a, ks in cases():
        out[f"{name}_rp"] = a.pattern.row_pointers
        out[f"{name}_ci"] = a.pattern.column_indices
        out[f"{name}_vals"] = a.values
        out[f"{name}_b"] = np.array(a.block_size)
        w = bs.transmissibility_weights(a)
        keys = sorted(w)
        out[f"{name}_wkeys"] = np.array(keys, dtype=np.int64).reshape(-1, 2)
        out[f"{name}_w"] = np.array([w[k] for k in keys])
        out[f"{name}_ks"] = np.array(ks)
        for k in ks:
            p = bs.partition(a.pattern, w, k)
            out[f"{name}_k{k}_part"] = p.cell_partition
            out[f"{name}_k{k}_cut"] = np.array(p.edge_cut_weight)
    np.savez_compressed(HERE / "partitions.npz", **out)
    print(sorted({k.split("_")[0] for k in out}))


if __name__ == "__main__":
    main()
