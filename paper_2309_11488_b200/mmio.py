"""System files (drop-in for bs/io.py:22-320): scalar coordinate Matrix
Market with a ``% blocksize: <b>`` comment, a ``<stem>_b.mtx`` array-format
right-hand side and a ``<stem>_wells.txt`` well file.

Same format, grouping rules and exceptions as the reference; the matrix body
is parsed by pandas' C tokenizer and grouped into blocks with array
operations instead of a per-line Python parse (the NORNE-size files of
SURVEY.md §8(f) row 3 have tens of millions of scalar lines).  With
``read_system(path, pinned=True)`` the matrix and vectors land in
page-locked host memory, ready for the solver's DMA upload.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np

from .blockcore import BlockMatrix, BlockVector, Layout, SparsityPattern
from .errors import BlockingError, DuplicateEntry, IndexOutOfRange, ParseError, ShapeError
from .synthetic import BundleMeta, SystemBundle
from .wells import MultisegmentWell, StandardWell, WellMode, WellSet

_MATRIX_HEADER = ("matrixmarket", "matrix", "coordinate", "real", "general")
_ARRAY_HEADER = ("matrixmarket", "matrix", "array", "real", "general")


def rhs_path(path) -> Path:
    p = Path(path)
    return p.with_name(p.stem + "_b.mtx")


def wells_path(path) -> Path:
    p = Path(path)
    return p.with_name(p.stem + "_wells.txt")


# ---------------------------------------------------------------------------
# writing (bs/io.py:62-121)

def _fmt(x: float) -> str:
    return repr(float(x))


def write_system(bundle, path) -> None:
    """Matrix to ``path`` plus ``<stem>_b.mtx`` / ``<stem>_wells.txt``."""
    a = bundle.a.as_block_row_major()
    b = a.block_size
    nb = a.num_block_rows
    n = nb * b
    p = a.pattern
    rows = np.repeat(np.arange(nb, dtype=np.int64), np.diff(p.row_pointers))
    li, lj = np.meshgrid(np.arange(b), np.arange(b), indexing="ij")
    si = (rows[:, None, None] * b + li[None] + 1).reshape(-1)
    sj = (p.column_indices[:, None, None] * b + lj[None] + 1).reshape(-1)
    vals = a.values.reshape(-1)
    body = "\n".join(f"{i} {j} {_fmt(v)}" for i, j, v in zip(si.tolist(), sj.tolist(),
                                                             vals.tolist()))
    head = ["%%MatrixMarket matrix coordinate real general", f"% blocksize: {b}",
            f"{n} {n} {p.num_blocks * b * b}"]
    Path(path).write_text("\n".join(head) + ("\n" + body if body else "") + "\n")
    rl = ["%%MatrixMarket matrix array real general", f"% blocksize: {b}", f"{n} 1"]
    rl.extend(_fmt(v) for v in bundle.rhs.data.tolist())
    rhs_path(path).write_text("\n".join(rl) + "\n")
    wells = getattr(bundle, "wells", None)
    if wells is not None and not wells.is_empty:
        wells_path(path).write_text(_format_wells(wells))
    elif wells_path(path).exists():
        wells_path(path).unlink()


def _format_wells(wells: WellSet) -> str:
    out = [f"mode {wells.mode.value}"]
    for w in wells.standard:
        m, n = w.block_dims
        out.append(f"well standard {m} {n} {len(w.perforated_cells)}")
        out.append("cells " + " ".join(str(int(c)) for c in w.perforated_cells))
        for tag, blocks in (("B", w.b_blocks), ("C", w.c_blocks)):
            for blk in blocks:
                out.append(f"{tag} " + " ".join(_fmt(v) for v in blk.reshape(-1)))
        out.append("Dinv " + " ".join(_fmt(v) for v in w.d_inverse.reshape(-1)))
    for w in wells.multisegment:
        m, n = w.block_dims
        out.append(f"well multisegment {m} {n} {w.nseg} {len(w.b_cells)} {len(w.c_cells)}")
        for tag, segs, cells, blocks in (("B", w.b_segments, w.b_cells, w.b_blocks),
                                         ("C", w.c_segments, w.c_cells, w.c_blocks)):
            for s, c, blk in zip(segs, cells, blocks):
                out.append(f"{tag} {int(s)} {int(c)} " + " ".join(_fmt(v) for v in blk.reshape(-1)))
        out.append("D " + " ".join(_fmt(v) for v in w.d_dense.reshape(-1)))
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------------------
# reading (bs/io.py:124-320)

def _split_header(text: str):
    """(header line, blocksize or None, lines, index of the first data line);
    ``text`` may be just the head of the file."""
    lines = text.splitlines()
    k = 0
    while k < len(lines) and not lines[k].strip():
        k += 1
    if k == len(lines) or not lines[k].strip().startswith("%%"):
        raise ParseError("missing MatrixMarket header")
    header = lines[k].strip()
    bsize = None
    k += 1
    while k < len(lines):
        line = lines[k].strip()
        if line and not line.startswith("%"):
            break
        body = line.lstrip("%").strip().lower()
        if bsize is None and body.startswith("blocksize:"):
            try:
                bsize = int(body.split(":", 1)[1])
            except ValueError:
                raise ParseError(f"bad blocksize comment {line!r}")
        k += 1
    return header, bsize, lines, k


def _head(p: Path, nbytes: int = 1 << 16) -> str:
    with open(p, "r") as fh:
        return fh.read(nbytes)


def _parse_header(line: str, want) -> None:
    if tuple(line.lstrip("%").lower().split()) != want:
        raise ParseError(f"unsupported header {line!r}")


def _parse_entries(p: Path, skip: int, nnz: int):
    """(rows, cols, values) of the coordinate body: the file after its first
    ``skip`` lines, tokenised by pandas' C parser (round-trip float parsing:
    values come back bit for bit)."""
    import pandas as pd
    try:
        df = pd.read_csv(p, sep=r"\s+", header=None, engine="c", skiprows=skip, comment="%",
                         float_precision="round_trip",
                         dtype={0: np.int64, 1: np.int64, 2: np.float64})
    except pd.errors.EmptyDataError:
        df = None
    except Exception:
        raise ParseError("malformed entry line")
    if df is None or len(df) == 0:
        if nnz:
            raise ParseError(f"expected {nnz} entries, found 0")
        return np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0)
    if df.shape[1] != 3 or df.isnull().values.any():
        raise ParseError("malformed entry line")
    if len(df) != nnz:
        raise ParseError(f"expected {nnz} entries, found {len(df)}")
    return (df[0].to_numpy(np.int64) - 1, df[1].to_numpy(np.int64) - 1,
            df[2].to_numpy(np.float64))


def _alloc(n, dtype, pinned):
    if pinned:
        from ._device import pinned_empty
        return pinned_empty(n, dtype)
    return np.empty(n, dtype=dtype)


def _read_matrix(p: Path, pinned: bool = False) -> BlockMatrix:
    header, b, lines, k = _split_header(_head(p))
    _parse_header(header, _MATRIX_HEADER)
    if b is None:
        raise ParseError("missing '% blocksize: <b>' comment")
    while k < len(lines) and not lines[k].strip():
        k += 1
    if k >= len(lines):
        raise ParseError("missing dimensions line")
    dims = lines[k].split()
    if len(dims) != 3:
        raise ParseError(f"bad dimensions line {lines[k]!r}")
    nrows, ncols, nnz = (int(t) for t in dims)
    if nrows != ncols:
        raise ParseError("matrix must be square")
    if nrows % b:
        raise BlockingError(f"{nrows} rows not divisible by block size {b}")
    nb = nrows // b
    si, sj, sv = _parse_entries(p, k + 1, nnz)
    if nnz == 0:
        pattern = SparsityPattern(nb, np.zeros(nb + 1, dtype=np.int64),
                                  np.empty(0, dtype=np.int64))
        return BlockMatrix(pattern, b, np.empty(0), Layout.BLOCK_ROW_MAJOR)
    if si.min() < 0 or sj.min() < 0 or si.max() >= nrows or sj.max() >= ncols:
        raise IndexOutOfRange("scalar coordinate outside the declared size")
    key_s = si * ncols + sj
    order = np.argsort(key_s, kind="stable")
    ks = key_s[order]
    if ks.size > 1:
        dup = np.flatnonzero(np.diff(ks) == 0)
        if dup.size:
            q = order[dup[0]]
            raise DuplicateEntry(f"scalar ({si[q] + 1}, {sj[q] + 1}) appears twice")
    bi, li = np.divmod(si, b)
    bj, lj = np.divmod(sj, b)
    key = bi * nb + bj
    uniq = np.unique(key)
    rows = uniq // nb
    rp = _alloc(nb + 1, np.int64, pinned)
    rp[0] = 0
    np.cumsum(np.bincount(rows, minlength=nb), out=rp[1:])
    ci = _alloc(uniq.size, np.int64, pinned)
    ci[:] = uniq % nb
    vals = _alloc(uniq.size * b * b, np.float64, pinned)
    vals[:] = 0.0
    v3 = vals.reshape(uniq.size, b, b)
    v3[np.searchsorted(uniq, key), li, lj] = sv
    return BlockMatrix(SparsityPattern(nb, rp, ci), b, vals, Layout.BLOCK_ROW_MAJOR)


def _read_rhs(p: Path, a: BlockMatrix, pinned: bool = False) -> BlockVector:
    header, _, lines, k = _split_header(p.read_text())
    _parse_header(header, _ARRAY_HEADER)
    while k < len(lines) and not lines[k].strip():
        k += 1
    if k >= len(lines):
        raise ParseError("missing dimensions line in rhs file")
    dims = lines[k].split()
    if len(dims) != 2 or int(dims[1]) != 1:
        raise ParseError("rhs must be a single column")
    n = int(dims[0])
    if n % a.block_size:
        raise BlockingError("rhs length not divisible by the block size")
    if n != a.num_block_rows * a.block_size:
        raise ShapeError("rhs length differs from the matrix")
    body = [ln for ln in lines[k + 1:] if ln.strip() and not ln.lstrip().startswith("%")]
    if len(body) != n:
        raise ParseError(f"expected {n} rhs values, found {len(body)}")
    try:
        data = np.array(body, dtype=np.float64) if n else np.zeros(0)
    except ValueError:
        raise ParseError("malformed rhs value")
    out = _alloc(n, np.float64, pinned)
    out[:] = data
    return BlockVector(out, a.block_size)


def _read_wells(p: Path) -> WellSet:
    lines = [ln.strip() for ln in p.read_text().splitlines() if ln.strip()]
    try:
        return _parse_wells(lines)
    except (ValueError, IndexError) as exc:
        raise ParseError(f"malformed well file: {exc}") from None


def _parse_wells(lines) -> WellSet:
    mode = WellMode.SEPARATE
    idx = 0
    if lines and lines[0].startswith("mode"):
        try:
            mode = WellMode(lines[0].split()[1])
        except (IndexError, ValueError):
            raise ParseError(f"bad mode line {lines[0]!r}")
        idx = 1
    standard, multisegment = [], []

    def floats(tag, line):
        parts = line.split()
        if parts[0] != tag:
            raise ParseError(f"expected {tag} record, found {line!r}")
        return np.array([float(t) for t in parts[1:]])

    while idx < len(lines):
        head = lines[idx].split()
        if head[0] != "well" or len(head) < 2:
            raise ParseError(f"expected well record, found {lines[idx]!r}")
        if head[1] == "standard":
            m, n, nperf = (int(t) for t in head[2:5])
            idx += 1
            cell_parts = lines[idx].split()
            if cell_parts[0] != "cells" or len(cell_parts) != nperf + 1:
                raise ParseError("bad cells record")
            cells = np.array([int(t) for t in cell_parts[1:]], dtype=np.int64)
            idx += 1
            bb = np.array([floats("B", lines[idx + q]) for q in range(nperf)])
            idx += nperf
            cc = np.array([floats("C", lines[idx + q]) for q in range(nperf)])
            idx += nperf
            dinv = floats("Dinv", lines[idx]).reshape(m, m)
            idx += 1
            standard.append(StandardWell(cells, bb.reshape(nperf, m, n), cc.reshape(nperf, m, n),
                                         dinv))
        elif head[1] == "multisegment":
            m, n, nseg, nb_e, nc_e = (int(t) for t in head[2:7])
            idx += 1

            def entries(tag, count, at):
                segs, cells, blocks = [], [], []
                for q in range(count):
                    parts = lines[at + q].split()
                    if parts[0] != tag:
                        raise ParseError(f"expected {tag} record")
                    segs.append(int(parts[1]))
                    cells.append(int(parts[2]))
                    blocks.append([float(t) for t in parts[3:]])
                return (np.array(segs, dtype=np.int64), np.array(cells, dtype=np.int64),
                        np.array(blocks).reshape(count, m, n))

            bs_, bc, bblk = entries("B", nb_e, idx)
            idx += nb_e
            cs, cc_, cblk = entries("C", nc_e, idx)
            idx += nc_e
            d = floats("D", lines[idx]).reshape(nseg * m, nseg * m)
            idx += 1
            multisegment.append(MultisegmentWell(nseg, bs_, bc, bblk, cs, cc_, cblk, d))
        else:
            raise ParseError(f"unknown well kind {head[1]!r}")
    return WellSet(standard, multisegment, mode)


def read_system(path, pinned: bool = False):
    """Read a system written by :func:`write_system` (bs/io.py:175-190):
    a missing rhs file yields zeros, missing wells an empty set."""
    p = Path(path)
    a = _read_matrix(p, pinned)
    rp = rhs_path(p)
    if rp.exists():
        rhs = _read_rhs(rp, a, pinned)
    else:
        rhs = BlockVector.zeros(a.num_block_rows, a.block_size)
    wp = wells_path(p)
    wells = _read_wells(wp) if wp.exists() else WellSet()
    return SystemBundle(a, rhs, wells, BundleMeta(name=p.stem, block_size=a.block_size))


__all__ = ["BundleMeta", "read_system", "write_system", "rhs_path", "wells_path"]
