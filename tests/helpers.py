"""Pattern / matrix builders shared by the tests (modelled on the reference's
conftest fixtures, bs tests/conftest.py:9-112)."""

import numpy as np


def pattern_from_rows(rows, n):
    from paper_2309_11488_b200 import SparsityPattern
    rp = np.zeros(n + 1, dtype=np.int64)
    cols = []
    for r in range(n):
        cs = sorted(set(rows.get(r, [])))
        rp[r + 1] = rp[r] + len(cs)
        cols.extend(cs)
    return SparsityPattern(n, rp, np.array(cols, dtype=np.int64))


def dominant_matrix(p, b, rng):
    from paper_2309_11488_b200 import BlockMatrix
    nnz = p.num_blocks
    vals = rng.uniform(-1.0, 1.0, size=(nnz, b, b))
    rows = np.repeat(np.arange(p.num_block_rows), np.diff(p.row_pointers))
    off = rows != p.column_indices
    sums = np.zeros((p.num_block_rows, b))
    np.add.at(sums, rows[off], np.abs(vals[off]).sum(axis=2))
    d = np.flatnonzero(~off)
    vals[d] = 0.0
    vals[d[:, None], np.arange(b)[None, :], np.arange(b)[None, :]] = sums[rows[d]] + 1.0
    return BlockMatrix(p, b, vals.reshape(-1))


def stencil_pattern(nx, ny, nz):
    n = nx * ny * nz
    rows = {i: [i] for i in range(n)}
    for i in range(n):
        ix, iy, iz = i % nx, (i // nx) % ny, i // (nx * ny)
        for ok, j in ((ix < nx - 1, i + 1), (iy < ny - 1, i + nx), (iz < nz - 1, i + nx * ny)):
            if ok:
                rows[i].append(j)
                rows[j].append(i)
    return pattern_from_rows(rows, n)
