"""The greedy partitioner (bs/jacobi.py:46-108) against the reference's own
output (tests/golden/make_partitions.py): edge weights bit for bit, the cell
assignment array-equal, the cut weight to rounding.  Host code (C++ walk in
libb200solve.so, no GPU needed)."""

import numpy as np
import pytest

import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import jacobi as J


def systems(golden):
    g = golden("partitions")
    names = sorted({k[: -len("_rp")] for k in g if k.endswith("_rp")})
    for name in names:
        rp, ci = g[f"{name}_rp"], g[f"{name}_ci"]
        a = P.BlockMatrix(P.SparsityPattern(len(rp) - 1, rp, ci), int(g[f"{name}_b"]),
                          g[f"{name}_vals"])
        yield name, a, g


def test_weights_bit_exact(golden):
    for name, a, g in systems(golden):
        w = P.transmissibility_weights(a)
        keys = sorted(w)
        np.testing.assert_array_equal(np.array(keys).reshape(-1, 2), g[f"{name}_wkeys"])
        np.testing.assert_array_equal(np.array([w[k] for k in keys]), g[f"{name}_w"])
        e = J._edge_weights(a)
        np.testing.assert_array_equal(np.stack([e.lo, e.hi], 1), g[f"{name}_wkeys"])
        np.testing.assert_array_equal(e.w, g[f"{name}_w"])


def test_partition_equals_reference(golden):
    for name, a, g in systems(golden):
        w = P.transmissibility_weights(a)
        for k in g[f"{name}_ks"]:
            k = int(k)
            ref = g[f"{name}_k{k}_part"]
            for weights in (w, J._edge_weights(a)):     # dict API and array fast path
                p = P.partition(a.pattern, weights, k)
                np.testing.assert_array_equal(p.cell_partition, ref, err_msg=f"{name} k={k}")
                np.testing.assert_allclose(p.edge_cut_weight, float(g[f"{name}_k{k}_cut"]),
                                           rtol=1e-12)


def test_partition_errors():
    a = P.generate(P.GeneratorSpec(3, 3, 2, seed=1)).a
    w = P.transmissibility_weights(a)
    with pytest.raises(P.TooManyPartitions):
        P.partition(a.pattern, w, a.num_block_rows + 1)
    with pytest.raises(ValueError):
        P.partition(a.pattern, w, 0)
    bad = dict(w)
    bad.pop(next(iter(bad)))
    with pytest.raises(ValueError):
        P.partition(a.pattern, bad, 2)
