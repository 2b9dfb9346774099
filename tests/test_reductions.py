"""The reference's chunk-64 inner product (bs/krylov.py:30-47) bit for bit.

CPU: the spelled-out summation order in oracle/port.py (the order
csrc/refdot.cu implements) equals numpy's np.add.reduceat + cumsum on this
host, over sizes that exercise every branch (empty, < 8 after the seed,
8-accumulator loop + tail, partial last chunk) and wide dynamic ranges.
GPU: the device kernel and the public dot/norm/dot_partials equal the
oracle bitwise."""

import numpy as np
import pytest

from oracle import port as O

SIZES = list(range(0, 140)) + [191, 192, 193, 1000, 4097, 65_536 + 7]


def _vectors(rng, m, wide):
    if wide:
        a = rng.standard_normal(m) * np.exp(rng.uniform(-30, 30, m))
    else:
        a = rng.uniform(-1.0, 1.0, m)
    return a, rng.standard_normal(m)


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("wide", [False, True])
def test_explicit_order_is_numpys(wide):
    rng = np.random.default_rng(5 + wide)
    for m in SIZES:
        a, b = _vectors(rng, m, wide)
        np.testing.assert_array_equal(_bits(O.dot_partials_explicit(a, b)),
                                      _bits(O.dot_partials(a, b)), err_msg=str(m))


def test_explicit_order_keeps_negative_zero():
    for m in (1, 3, 9, 64, 70):
        z = -np.zeros(m)
        assert np.all(np.signbit(O.dot_partials_explicit(z, np.ones(m))))
        assert np.all(np.signbit(O.dot_partials(z, np.ones(m))))


@pytest.mark.gpu
@pytest.mark.parametrize("wide", [False, True])
def test_device_chunked_dot_bit_exact(wide):
    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200 import krylov as K
    rng = np.random.default_rng(11 + wide)
    for m in SIZES + [3_000_000]:
        a, b = _vectors(rng, m, wide)
        np.testing.assert_array_equal(_bits(K.dot_partials(a, b)), _bits(O.dot_partials(a, b)),
                                      err_msg=str(m))
        assert _bits(K.dot_arrays(a, b)) == _bits(O.dot(a, b)), m
        assert _bits(K.norm_array(a)) == _bits(O.norm(a)), m
        if m % 3 == 0 and m:
            va, vb = P.BlockVector(a, 3), P.BlockVector(b, 3)
            assert _bits(P.dot(va, vb)) == _bits(O.dot(a, b))
            assert _bits(P.norm(va)) == _bits(O.norm(a))


@pytest.mark.gpu
def test_reported_initial_norm_is_reference_order():
    """solve_with_fallback / bicgstab report norm_array(b - A x0) exactly
    (bs/krylov.py:175-176), with and without an initial guess, on both the
    native device loop and the well-augmented loop."""
    import paper_2309_11488_b200 as P
    from paper_2309_11488_b200.krylov import norm_array
    g = P.generate(P.GeneratorSpec(9, 8, 7, seed=3))
    rng = np.random.default_rng(2)
    x0 = P.BlockVector(rng.uniform(-1, 1, g.rhs.data.size), 3)
    for backend in P.Backend:
        cfg = P.SolverConfig(backend=backend, stop=P.StoppingCriteria(1e-6, 200))
        _, rep = P.solve_with_fallback(cfg, g.a, g.rhs)
        assert rep.initial_norm == norm_array(g.rhs.data)
        _, rep = P.solve_with_fallback(cfg, g.a, g.rhs, x0=x0)
        assert rep.initial_norm == norm_array(g.rhs.data - P.spmv(g.a, x0).data)
    fact = P.decompose(g.a, P.graph_color(g.a.pattern))
    _, rep = P.bicgstab(P.MatrixOperator(g.a), fact, g.rhs, x0=x0)
    assert rep.initial_norm == norm_array(g.rhs.data - P.spmv(g.a, x0).data)
    _, rep = P.bicgstab(P.MatrixOperator(g.a), fact, g.rhs)
    assert rep.initial_norm == norm_array(g.rhs.data)
