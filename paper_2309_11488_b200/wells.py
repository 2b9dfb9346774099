"""Well operators (drop-in for bs/wells.py): standard and multi-segment wells
applied separately after each SpMV on the GPU, or folded into the matrix
(coupled mode, host-side as in the reference).

Separate application (``WellAugmentedOperator``, bs/krylov.py:84-94) runs in
csrc/wells.cu: one warp per well forms t2 = D^-1 (B x) (standard: stored
inverse; multi-segment: the pivoted dense LU factors from scipy's
``lu_factor``, exactly the factors the reference keeps), then one thread per
perforated cell subtracts C^T t2 for that cell's wells in the reference's
order.  ``fold_into_matrix`` (bs/wells.py:218-283) stays on the host: it is
one-off assembly, not part of the iteration.
"""

from __future__ import annotations

import ctypes as C
import enum
import hashlib
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch
from scipy.linalg import lu_factor, lu_solve

from . import _device as D
from ._lib import check
from .blockcore import BlockMatrix, BlockVector, Layout, SparsityPattern
from .errors import ShapeError, SingularWellMatrix


class WellMode(enum.Enum):
    COUPLED = "coupled"
    SEPARATE = "separate"


@dataclass
class StandardWell:
    """One MxN block of B and C per perforation plus the stored D inverse
    (bs/wells.py:29-57)."""

    perforated_cells: np.ndarray
    b_blocks: np.ndarray
    c_blocks: np.ndarray
    d_inverse: np.ndarray

    def __post_init__(self):
        self.perforated_cells = np.asarray(self.perforated_cells, dtype=np.int64)
        self.b_blocks = np.asarray(self.b_blocks, dtype=np.float64)
        self.c_blocks = np.asarray(self.c_blocks, dtype=np.float64)
        self.d_inverse = np.asarray(self.d_inverse, dtype=np.float64)
        p = len(self.perforated_cells)
        if p == 0:
            raise ShapeError("a well needs at least one perforation")
        if np.any(np.diff(self.perforated_cells) <= 0):
            raise ShapeError("perforated cells must be strictly increasing")
        m, n = self.block_dims
        if self.b_blocks.shape != (p, m, n) or self.c_blocks.shape != (p, m, n):
            raise ShapeError("B/C blocks must be (perforations, M, N)")
        if self.d_inverse.shape != (m, m) or not np.all(np.isfinite(self.d_inverse)):
            raise ShapeError("D inverse must be a finite MxM block")

    @property
    def block_dims(self) -> tuple[int, int]:
        return self.d_inverse.shape[0], self.b_blocks.shape[2]


@dataclass
class MultisegmentWell:
    """Segmented well: sparse per-segment B/C, dense D with its pivoted LU
    factors computed once per value update (bs/wells.py:60-122)."""

    nseg: int
    b_segments: np.ndarray
    b_cells: np.ndarray
    b_blocks: np.ndarray
    c_segments: np.ndarray
    c_cells: np.ndarray
    c_blocks: np.ndarray
    d_dense: np.ndarray
    _d_factors: tuple = field(repr=False, default=None)

    def __post_init__(self):
        self.b_segments = np.asarray(self.b_segments, dtype=np.int64)
        self.b_cells = np.asarray(self.b_cells, dtype=np.int64)
        self.b_blocks = np.asarray(self.b_blocks, dtype=np.float64)
        self.c_segments = np.asarray(self.c_segments, dtype=np.int64)
        self.c_cells = np.asarray(self.c_cells, dtype=np.int64)
        self.c_blocks = np.asarray(self.c_blocks, dtype=np.float64)
        self.d_dense = np.asarray(self.d_dense, dtype=np.float64)
        m, n = self.block_dims
        for seg, cells, blocks, name in ((self.b_segments, self.b_cells, self.b_blocks, "B"),
                                         (self.c_segments, self.c_cells, self.c_blocks, "C")):
            if blocks.shape != (len(seg), m, n) or len(cells) != len(seg):
                raise ShapeError(f"{name} entries must be (segment, cell, MxN block)")
            if len(np.unique(cells)) != len(cells):
                raise ShapeError(f"columns of {name} may hold at most one block")
            if len(seg) and (seg.min() < 0 or seg.max() >= self.nseg):
                raise ShapeError(f"{name} segment index outside [0, nseg)")
        size = self.nseg * m
        if self.d_dense.shape != (size, size):
            raise ShapeError("D must be dense (nseg*M, nseg*M)")
        self._refactor()

    def _refactor(self):
        if not np.all(np.isfinite(self.d_dense)):
            raise SingularWellMatrix("well matrix D contains non-finite entries")
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            lu, piv = lu_factor(self.d_dense, check_finite=False)
        if np.any(np.diag(lu) == 0.0) or not np.all(np.isfinite(lu)):
            raise SingularWellMatrix("well matrix D admits no LU factorization")
        self._d_factors = (lu, piv)

    @property
    def block_dims(self) -> tuple[int, int]:
        m = self.d_dense.shape[0] // self.nseg
        return m, self.b_blocks.shape[2] if self.b_blocks.ndim == 3 else 0

    def solve_d(self, rhs: np.ndarray) -> np.ndarray:
        return lu_solve(self._d_factors, rhs, check_finite=False)


def _check_cells(cells: np.ndarray, num_blocks: int):
    if len(cells) and (cells.min() < 0 or cells.max() >= num_blocks):
        raise ShapeError("well perforates a cell outside the matrix")


class _WellsArgs(C.Structure):
    _P = C.c_void_p
    _fields_ = [("nwells", C.c_int), ("nb", C.c_int), ("kind", _P), ("M", _P), ("nseg", _P),
                ("bptr", _P), ("bcell", _P), ("bseg", _P), ("boff", _P), ("bvals", _P),
                ("doff", _P), ("dvals", _P), ("pivoff", _P), ("piv", _P), ("toff", _P),
                ("ncells", C.c_int), ("cells", _P), ("cptr", _P), ("ccoff", _P), ("ct2", _P),
                ("cM", _P), ("cvals", _P)]


class DeviceWells:
    """A WellSet packed for csrc/wells.cu (standard wells first, then
    multi-segment ones; C entries grouped by cell in that well order)."""

    def __init__(self, wells: "WellSet", nb: int, num_cells: int):
        dev = D.require_cuda()
        order = [(0, w) for w in wells.standard] + [(1, w) for w in wells.multisegment]
        kind, Ms, nseg, bptr, bcell, bseg, boff, bvals = [], [], [], [0], [], [], [], []
        doff, dvals, pivoff, piv, toff = [], [], [], [], []
        centries = []   # (cell, well order, C block, t2 offset, M)
        dpos = ppos = tpos = bpos = 0
        for wi, (k, w) in enumerate(order):
            m, n = w.block_dims
            if n != nb:
                raise ShapeError("well block width does not match the matrix")
            if k == 0:
                _check_cells(w.perforated_cells, num_cells)
                cells_b, segs_b, blocks_b = w.perforated_cells, np.zeros(len(w.perforated_cells), np.int64), w.b_blocks
                cells_c, segs_c, blocks_c = w.perforated_cells, segs_b, w.c_blocks
                d = w.d_inverse.reshape(-1)
                s = 1
            else:
                _check_cells(w.b_cells, num_cells)
                _check_cells(w.c_cells, num_cells)
                cells_b, segs_b, blocks_b = w.b_cells, w.b_segments, w.b_blocks
                cells_c, segs_c, blocks_c = w.c_cells, w.c_segments, w.c_blocks
                lu, pv = w._d_factors
                d = np.ascontiguousarray(lu).reshape(-1)
                piv.append(np.asarray(pv, dtype=np.int32))
                s = w.nseg
            if m > 32 or s * m > 32 * 64:
                raise ShapeError("well too large for the device well kernels")
            kind.append(k); Ms.append(m); nseg.append(s)
            for e in range(len(cells_b)):
                bcell.append(int(cells_b[e])); bseg.append(int(segs_b[e]))
                boff.append(bpos); bvals.append(blocks_b[e].reshape(-1)); bpos += m * n
            bptr.append(len(bcell))
            doff.append(dpos); dvals.append(d); dpos += d.size
            pivoff.append(ppos); ppos += (s * m if k == 1 else 0)
            toff.append(tpos)
            for e in range(len(cells_c)):
                centries.append((int(cells_c[e]), wi, blocks_c[e].reshape(-1),
                                 tpos + int(segs_c[e]) * m, m))
            tpos += s * m
        centries.sort(key=lambda t: (t[0], t[1]))   # per cell, in well order
        cells = sorted({c[0] for c in centries})
        cptr = np.searchsorted([c[0] for c in centries], cells + [num_cells + 1]).tolist() \
            if centries else [0]
        cvals, ccoff, ct2, cM, cpos = [], [], [], [], 0
        for c in centries:
            ccoff.append(cpos); cvals.append(c[2]); cpos += c[2].size
            ct2.append(c[3]); cM.append(c[4])

        def i32(v):
            return torch.tensor(np.asarray(v, dtype=np.int32).reshape(-1) if len(v) else
                                np.zeros(1, np.int32), device=dev)

        def i64(v):
            return torch.tensor(np.asarray(v, dtype=np.int64).reshape(-1) if len(v) else
                                np.zeros(1, np.int64), device=dev)

        def f64(parts):
            a = np.concatenate(parts) if parts else np.zeros(1)
            return torch.tensor(a, dtype=torch.float64, device=dev)

        self._t = dict(kind=i32(kind), M=i32(Ms), nseg=i32(nseg), bptr=i32(bptr),
                       bcell=i32(bcell), bseg=i32(bseg), boff=i64(boff), bvals=f64(bvals),
                       doff=i64(doff), dvals=f64(dvals), pivoff=i64(pivoff),
                       piv=i32(np.concatenate(piv) if piv else []), toff=i64(toff),
                       cells=i32(cells), cptr=i32(cptr), ccoff=i64(ccoff), ct2=i64(ct2),
                       cM=i32(cM), cvals=f64(cvals))
        self.nwells = len(order)
        self.nb = nb
        self.scratch = torch.empty(max(tpos, 1), dtype=torch.float64, device=dev)
        a = _WellsArgs()
        a.nwells, a.nb, a.ncells = self.nwells, nb, len(cells)
        for k, v in self._t.items():
            setattr(a, k, v.data_ptr())
        self._args = a

    def in_plan_order(self, perm: torch.Tensor, smap) -> "DeviceWells":
        """The same wells for device vectors in a plan's row order (perm: old
        row -> plan row, device): the cell indices are remapped on the device
        and the WellFix tables of the Krylov loop (csrc/sell.cuh) are built
        there too -- no host round trip.  Compact cell q keeps its input-order
        place; slice_tab[s] = 32 s when slice s holds a perforated row (else
        -1), lane_tab[32 s + lane] = its compact cell (else -1)."""
        out = DeviceWells.__new__(DeviceWells)
        out.__dict__.update(self.__dict__)
        dev = self.scratch.device
        perm = perm.to(torch.int64)
        t = dict(self._t)
        if self.nwells:
            t["bcell"] = perm.index_select(0, self._t["bcell"].long()).to(torch.int32)
            t["cells"] = perm.index_select(0, self._t["cells"].long()).to(torch.int32)
        out._t = t
        a = _WellsArgs()
        a.nwells, a.nb, a.ncells = self.nwells, self.nb, self._args.ncells
        for k, v in t.items():
            setattr(a, k, v.data_ptr())
        out._args = a
        ns = smap.nslices
        slice_tab = torch.full((max(ns, 1),), -1, dtype=torch.int32, device=dev)
        lane_tab = torch.full((max(32 * ns, 1),), -1, dtype=torch.int32, device=dev)
        nc = self._args.ncells
        if self.nwells and nc:
            rows = t["cells"][:nc].long()
            row0 = smap.row0[:ns].long()
            sl = torch.searchsorted(row0, rows, right=True) - 1
            lane = rows - row0.index_select(0, sl)
            slice_tab[sl] = (32 * sl).to(torch.int32)
            lane_tab[32 * sl + lane] = torch.arange(nc, dtype=torch.int32, device=dev)
        corr = torch.empty(max(nc * self.nb, 1), dtype=torch.float64, device=dev)
        out.tables = (slice_tab, lane_tab, corr)
        return out

    def apply(self, x: torch.Tensor, y: torch.Tensor):
        """y -= sum of the wells' C^T D^-1 B x (device vectors, input order)."""
        if self.nwells:
            check(D.lib().b2s_wells_apply(C.byref(self._args), D.ptr(x), D.ptr(y),
                                          D.ptr(self.scratch), D.stream()), "wells_apply")


@dataclass
class WellSet:
    """All wells of one system plus the coupled/separate handling mode
    (bs/wells.py:165-202)."""

    standard: list = field(default_factory=list)
    multisegment: list = field(default_factory=list)
    mode: WellMode = WellMode.SEPARATE

    @property
    def is_empty(self) -> bool:
        return not self.standard and not self.multisegment

    def _fingerprint(self) -> bytes:
        """Digest of every host array of every well (the reference reads them
        at each apply, bs/wells.py:125-162): a device copy is reused only
        while the wells are unchanged -- values updated in place (e.g.
        d_dense plus _refactor), wells appended or removed."""
        h = hashlib.blake2b(digest_size=16)
        for w in (*self.standard, None, *self.multisegment):
            if w is None:
                h.update(b"|")
                continue
            for k, v in sorted(vars(w).items()):
                for j, arr in enumerate(v if isinstance(v, tuple) else (v,)):
                    if isinstance(arr, np.ndarray):
                        h.update(f"{k}{j}{arr.dtype.str}{arr.shape}".encode())
                        h.update(np.ascontiguousarray(arr).tobytes())
        return h.digest()

    def device(self, nb: int, num_cells: int) -> DeviceWells:
        key = (nb, num_cells)
        cache = self.__dict__.setdefault("_dev", {})
        fp = self._fingerprint()
        hit = cache.get(key)
        if hit is None or hit[0] != fp:
            hit = cache[key] = (fp, DeviceWells(self, nb, num_cells))
        return hit[1]

    def apply_contributions(self, x: BlockVector, y: BlockVector) -> BlockVector:
        if self.mode is WellMode.COUPLED:
            return y
        self.apply_contributions_array(x.data, y.data, x.block_size)
        return y

    def apply_contributions_array(self, x: np.ndarray, y: np.ndarray, n: int):
        """In place on host arrays (computed on the device)."""
        if self.mode is WellMode.COUPLED or self.is_empty:
            return
        dev = D.require_cuda()
        dw = self.device(n, y.size // n)
        xd, yd = D.f64(x, dev), D.f64(y, dev)
        dw.apply(xd, yd)
        y[:] = yd.cpu().numpy()


def apply_standard(w: StandardWell, x: BlockVector, y: BlockVector) -> BlockVector:
    """In place: y -= C^T (D^-1 (B x)) (bs/wells.py:125-132)."""
    m, n = w.block_dims
    if x.block_size != n or y.block_size != n or x.num_blocks != y.num_blocks:
        raise ShapeError("vector block size does not match the well")
    _check_cells(w.perforated_cells, x.num_blocks)
    WellSet([w]).apply_contributions_array(x.data, y.data, n)
    return y


def apply_multisegment(w: MultisegmentWell, x: BlockVector, y: BlockVector) -> BlockVector:
    """In place: y -= C^T (D^-1 (B x)), D through its LU (bs/wells.py:143-151)."""
    m, n = w.block_dims
    if x.block_size != n or y.block_size != n or x.num_blocks != y.num_blocks:
        raise ShapeError("vector block size does not match the well")
    _check_cells(w.b_cells, x.num_blocks)
    _check_cells(w.c_cells, x.num_blocks)
    WellSet([], [w]).apply_contributions_array(x.data, y.data, n)
    return y


def fold_into_matrix(a: BlockMatrix, wells: WellSet) -> BlockMatrix:
    """A' = A - sum over wells of C^T D^-1 B with the pattern widened by every
    (row, col) pair of cells one well couples (bs/wells.py:218-283); host-side
    assembly, vectorised."""
    a = a.as_block_row_major()
    b, nb = a.block_size, a.num_block_rows
    rows_x, cols_x, deltas = [], [], []
    for w in wells.standard:
        _check_cells(w.perforated_cells, nb)
        if w.block_dims[1] != b:
            raise ShapeError("well block width does not match the matrix")
        t = np.einsum("ij,pjn->pin", w.d_inverse, w.b_blocks)          # D^-1 B_j
        d = np.einsum("ima,jmc->ijac", w.c_blocks, t)                   # C_i^T (D^-1 B_j)
        cells = w.perforated_cells
        rows_x.append(np.repeat(cells, len(cells)))
        cols_x.append(np.tile(cells, len(cells)))
        deltas.append(d.reshape(-1, b, b))
    for w in wells.multisegment:
        _check_cells(w.b_cells, nb)
        _check_cells(w.c_cells, nb)
        m, n = w.block_dims
        if n != b:
            raise ShapeError("well block width does not match the matrix")
        ne = len(w.b_cells)
        bdense = np.zeros((w.nseg * m, ne * n))
        for t_idx in range(ne):
            s = int(w.b_segments[t_idx])
            bdense[s * m:(s + 1) * m, t_idx * n:(t_idx + 1) * n] = w.b_blocks[t_idx]
        z = w.solve_d(bdense).reshape(w.nseg, m, ne, n)
        zc = z[w.c_segments]                                            # (nc, m, ne, n)
        d = np.einsum("cma,cmtn->ctan", w.c_blocks, zc)
        rows_x.append(np.repeat(w.c_cells, ne))
        cols_x.append(np.tile(w.b_cells, len(w.c_cells)))
        deltas.append(d.reshape(-1, b, b))
    p = a.pattern
    rows = np.repeat(np.arange(nb, dtype=np.int64), np.diff(p.row_pointers))
    if rows_x:
        allr = np.concatenate([rows, *rows_x])
        allc = np.concatenate([p.column_indices, *cols_x])
    else:
        allr, allc = rows, p.column_indices
    key = np.unique(allr * nb + allc)
    nr, nc = key // nb, key % nb
    rp = np.zeros(nb + 1, dtype=np.int64)
    np.cumsum(np.bincount(nr, minlength=nb), out=rp[1:])
    pat = SparsityPattern(nb, rp, nc)
    vals = np.zeros((key.size, b, b))
    vals[np.searchsorted(key, rows * nb + p.column_indices)] = a.values3d
    # subtract every well term in the reference's order (wells in list order)
    for rr, cc, dd in zip(rows_x, cols_x, deltas):
        np.subtract.at(vals, np.searchsorted(key, rr * nb + cc), dd)   # in order
    return BlockMatrix(pat, b, vals.reshape(-1), Layout.BLOCK_ROW_MAJOR)


__all__ = ["WellMode", "StandardWell", "MultisegmentWell", "WellSet", "DeviceWells",
           "apply_standard", "apply_multisegment", "fold_into_matrix"]
