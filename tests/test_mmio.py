"""System files (bs/io.py:22-320): reading what the reference wrote, round
trips, scalar grouping and the reference's parse errors (modelled on the
reference's tests/test_io.py).  CPU only."""

import numpy as np
import pytest
from numpy.testing import assert_array_equal

import paper_2309_11488_b200 as P
from paper_2309_11488_b200.mmio import rhs_path, wells_path

GOLDEN_MM = __import__("pathlib").Path(__file__).resolve().parent / "golden" / "mm"


@pytest.mark.parametrize("name,spec", [
    ("std", dict(nx=3, ny=2, nz=2, well_count=1, well_depth=2, seed=44)),
    ("msw", dict(nx=3, ny=3, nz=3, well_count=2, well_depth=3, well_kind="multisegment", seed=9)),
    ("b2", dict(nx=4, ny=3, nz=2, block_size=2, seed=7))])
def test_reads_reference_written_files(name, spec):
    back = P.read_system(GOLDEN_MM / f"{name}.mtx")
    src = P.generate(P.GeneratorSpec(**spec))
    assert_array_equal(back.a.pattern.row_pointers, src.a.pattern.row_pointers)
    assert_array_equal(back.a.pattern.column_indices, src.a.pattern.column_indices)
    assert_array_equal(back.a.values, src.a.values)
    assert_array_equal(back.rhs.data, src.rhs.data)
    for w0, w1 in zip(src.wells.standard, back.wells.standard):
        assert_array_equal(w1.perforated_cells, w0.perforated_cells)
        assert_array_equal(w1.b_blocks, w0.b_blocks)
        assert_array_equal(w1.d_inverse, w0.d_inverse)
    for w0, w1 in zip(src.wells.multisegment, back.wells.multisegment):
        assert w1.nseg == w0.nseg
        assert_array_equal(w1.b_cells, w0.b_cells)
        assert_array_equal(w1.d_dense, w0.d_dense)


def test_round_trip_bit_exact_and_mode(tmp_path):
    src = P.generate(P.GeneratorSpec(3, 2, 2, well_count=1, well_depth=2, seed=44))
    src.wells.mode = P.WellMode.COUPLED
    path = tmp_path / "case.mtx"
    P.write_system(src, path)
    back = P.read_system(path)
    assert_array_equal(back.a.values, src.a.values)
    assert_array_equal(back.rhs.data, src.rhs.data)
    assert back.wells.mode is P.WellMode.COUPLED
    assert rhs_path(path).name == "case_b.mtx" and wells_path(path).name == "case_wells.txt"
    rhs_path(path).unlink()
    wells_path(path).unlink()
    back = P.read_system(path)
    assert_array_equal(back.rhs.data, np.zeros_like(src.rhs.data))
    assert back.wells.is_empty


def test_scalar_grouping(tmp_path):
    path = tmp_path / "one.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real general\n% blocksize: 3\n"
                    "6 6 1\n2 2 5.0\n")
    a = P.read_system(path).a
    assert a.num_block_rows == 2 and a.pattern.num_blocks == 1
    want = np.zeros((3, 3))
    want[1, 1] = 5.0
    assert_array_equal(a.block(0, 0), want)
    nb = 44431
    path.write_text("%%MatrixMarket matrix coordinate real general\n% blocksize: 3\n"
                    f"{nb * 3} {nb * 3} 2\n1 1 1.0\n{nb * 3} {nb * 3} 2.0\n")
    a = P.read_system(path).a
    assert a.num_block_rows == nb and a.pattern.num_blocks == 2


@pytest.mark.parametrize("text,exc", [
    ("%%MatrixMarket matrix coordinate real general\n% blocksize: 1\n2 2 2\n1 1 1.0\n1 1 2.0\n",
     P.DuplicateEntry),
    ("%%MatrixMarket matrix array real general\n% blocksize: 1\n1 1 1\n1 1 0.5\n", P.ParseError),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n", P.ParseError),
    ("%%MatrixMarket matrix coordinate real general\n% blocksize: 3\n7 7 1\n1 1 1.0\n",
     P.BlockingError),
    ("%%MatrixMarket matrix coordinate real general\n% blocksize: 1\n2 2 3\n1 1 1.0\n",
     P.ParseError),
    ("%%MatrixMarket matrix coordinate real general\n% blocksize: 1\n2 2 1\n3 1 1.0\n",
     P.IndexOutOfRange),
])
def test_parse_errors(tmp_path, text, exc):
    path = tmp_path / "bad.mtx"
    path.write_text(text)
    with pytest.raises(exc):
        P.read_system(path)


@pytest.mark.gpu
def test_pinned_read_solves(tmp_path):
    """read_system(pinned=True) hands the solver page-locked buffers."""
    src = P.generate(P.GeneratorSpec(6, 5, 4, seed=3))
    path = tmp_path / "s.mtx"
    P.write_system(src, path)
    back = P.read_system(path, pinned=True)
    import torch
    assert torch.from_numpy(back.a.values).is_pinned()
    x, rep = P.solve_with_fallback(P.SolverConfig(), back.a, back.rhs)
    x0, rep0 = P.solve_with_fallback(P.SolverConfig(), src.a, src.rhs)
    assert rep.iterations == rep0.iterations
    assert_array_equal(x.data, x0.data)
