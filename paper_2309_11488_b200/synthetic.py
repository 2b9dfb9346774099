"""Synthetic reservoir-style block systems: the benchmark's input source.

``generate(GeneratorSpec(...))`` draws exactly the same random numbers in the
same order as the reference generator (``bs/io.py:363-414``), so a seed gives
the identical matrix and right-hand side: a 7-point stencil on an
``nx*ny*nz`` grid in natural order ``cell = ix + nx*(iy + ny*iz)``, every
off-diagonal block ``-t * U(0.5, 1.5)`` with the per-direction
transmissibility ``t``, each diagonal block ``diag(row abs sums) + boost*I``,
and a ``U(-1, 1)`` right-hand side, then the optional wells
(``bs/io.py:417-442``, same draws).

Two harness extensions build the BASELINE configs the reference generator
cannot express:

* ``generate_masked`` -- C2: a seeded inactive-cell mask (smoothed Gaussian
  field thresholded to an active fraction); couplings only between active
  cells, active cells renumbered in natural order, same value recipe.
* ``generate_heterogeneous`` -- C3: lognormal permeability ``k = exp(sigma*g)``
  with harmonic-mean face transmissibilities (ill-conditioned).

All three return host numpy arrays ``(rp, ci, vals3, rhs)`` wrapped in a
:class:`SystemBundle`; the input is resident on the host, like the
reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .blockcore import BlockMatrix, BlockVector, Layout, SparsityPattern
from .errors import ShapeError


@dataclass(frozen=True)
class GeneratorSpec:
    """Mirror of ``bs/io.py:326-360`` (defaults and validation)."""

    nx: int
    ny: int
    nz: int
    block_size: int = 3
    tx: float = 1.0
    ty: float = 1.0
    tz: float = 0.5
    diagonal_boost: float = 1.0
    well_count: int = 0
    well_kind: str = "standard"
    well_depth: int = 3
    seed: int = 0

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("grid dimensions must be >= 1")
        if self.diagonal_boost <= 0:
            raise ValueError("diagonal_boost must be positive")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")
        if self.well_kind not in ("standard", "multisegment"):
            raise ValueError("well_kind must be standard or multisegment")
        if self.well_count < 0 or (self.well_count and self.well_depth < 1):
            raise ValueError("wells need a non-negative count and depth >= 1")


@dataclass
class BundleMeta:
    """bs/io.py:27-31."""

    name: str
    block_size: int
    grid_dims: tuple | None = None


@dataclass
class SystemBundle:
    """bs/io.py:33-44: same fields, order and shape checks."""

    a: BlockMatrix
    rhs: BlockVector
    wells: object          # WellSet
    meta: BundleMeta

    def __post_init__(self):
        if self.rhs.block_size != self.a.block_size:
            raise ShapeError("rhs block size differs from the matrix")
        if self.rhs.num_blocks != self.a.num_block_rows:
            raise ShapeError("rhs length differs from the matrix")


def _faces(nx, ny, nz, active=None):
    """Face pairs (lo, hi) in the reference's order: all +x faces, then +y,
    then +z, each in ascending lower-cell order (bs/io.py:370-382)."""
    # the reference enumerates cells through meshgrid(..., indexing="ij"),
    # i.e. ix slowest and iz fastest; the random draws follow that order
    ix, iy, iz = (a.reshape(-1) for a in np.meshgrid(
        np.arange(nx, dtype=np.int64), np.arange(ny, dtype=np.int64),
        np.arange(nz, dtype=np.int64), indexing="ij"))
    cell = ix + nx * (iy + ny * iz)
    out = []
    for ok, step in ((ix < nx - 1, 1), (iy < ny - 1, nx), (iz < nz - 1, nx * ny)):
        lo = cell[ok]
        hi = lo + step
        if active is not None:
            keep = active[lo] & active[hi]
            lo, hi = lo[keep], hi[keep]
        out.append((lo, hi))
    return out


def _assemble(n, lo, hi, tvals, b, boost, rng):
    """Blocks for the 2*npairs directed couplings + n diagonals, sorted to
    BSR, diagonal = diag(scalar row abs sums) + boost*I (bs/io.py:384-408)."""
    npairs = lo.size
    src = np.concatenate([lo, hi, np.arange(n, dtype=np.int64)])
    dst = np.concatenate([hi, lo, np.arange(n, dtype=np.int64)])
    blk = np.empty((src.size, b, b))
    # one draw of 2*npairs*b*b uniforms, in directed-coupling order
    u = rng.uniform(0.5, 1.5, size=(2 * npairs, b, b))
    t2 = np.concatenate([tvals, tvals])
    blk[:2 * npairs] = -t2[:, None, None] * u
    blk[2 * npairs:] = 0.0
    order = np.lexsort((dst, src))
    src, dst, blk = src[order], dst[order], blk[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=rp[1:])
    sums = np.zeros((n, b))
    np.add.at(sums, src, np.abs(blk).sum(axis=2))
    diag = np.flatnonzero(src == dst)
    eye = np.arange(b)
    d = np.zeros((n, b, b))
    d[:, eye, eye] = sums + boost
    blk[diag] = d
    return rp, dst, blk


def _bundle(rp, ci, blk, rhs, b, name, dims, wells=None):
    from .wells import WellSet
    n = rp.size - 1
    pat = SparsityPattern(n, rp, ci)
    a = BlockMatrix(pat, b, blk.reshape(-1), Layout.BLOCK_ROW_MAJOR)
    return SystemBundle(a, BlockVector(rhs, b), WellSet() if wells is None else wells,
                        BundleMeta(name, b, dims))


def generate(spec: GeneratorSpec) -> SystemBundle:
    """Deterministic 7-point system, draw-for-draw identical to bs/io.py:363-414."""
    nx, ny, nz, b = spec.nx, spec.ny, spec.nz, spec.block_size
    n = nx * ny * nz
    rng = np.random.default_rng(spec.seed)
    faces = _faces(nx, ny, nz)
    lo = np.concatenate([f[0] for f in faces])
    hi = np.concatenate([f[1] for f in faces])
    t = np.concatenate([np.full(f[0].size, tv) for f, tv in
                        zip(faces, (spec.tx, spec.ty, spec.tz))])
    rp, ci, blk = _assemble(n, lo, hi, t, b, spec.diagonal_boost, rng)
    rhs = rng.uniform(-1.0, 1.0, size=n * b)
    wells = _generate_wells(spec, rng)
    return _bundle(rp, ci, blk, rhs, b, f"synthetic-{nx}x{ny}x{nz}", (nx, ny, nz), wells)


def _generate_wells(spec: GeneratorSpec, rng):
    """Vertical wells in random columns, same draws as bs/io.py:417-442."""
    from .wells import MultisegmentWell, StandardWell, WellSet
    if spec.well_count == 0:
        return WellSet()
    nx, ny, nz, b = spec.nx, spec.ny, spec.nz, spec.block_size
    depth = min(spec.well_depth, nz)
    m = b + 1
    columns = rng.choice(nx * ny, size=min(spec.well_count, nx * ny), replace=False)
    standard, multisegment = [], []
    for col in columns:
        cx, cy = int(col) % nx, int(col) // nx
        cells = np.array([cx + nx * (cy + ny * z) for z in range(depth)], dtype=np.int64)
        bb = rng.uniform(-0.1, 0.1, size=(depth, m, b))
        cc = rng.uniform(-0.1, 0.1, size=(depth, m, b))
        if spec.well_kind == "standard":
            d = np.eye(m) + rng.uniform(0.0, 0.1, size=(m, m)) / m
            standard.append(StandardWell(cells, bb, cc, np.linalg.inv(d)))
        else:
            size = depth * m
            d = np.eye(size) + rng.uniform(0.0, 0.5, size=(size, size)) / size
            seg = np.arange(depth, dtype=np.int64)
            multisegment.append(MultisegmentWell(depth, seg, cells, bb, seg.copy(), cells.copy(),
                                                 cc, d))
    return WellSet(standard, multisegment)


def _smooth_field(shape, sigma, rng):
    """Seeded N(0,1) field smoothed by a separable Gaussian (numpy only)."""
    g = rng.standard_normal(shape)
    for axis, s in enumerate(sigma):
        if s <= 0:
            continue
        r = int(np.ceil(3 * s))
        k = np.exp(-0.5 * (np.arange(-r, r + 1) / s) ** 2)
        k /= k.sum()
        g = np.apply_along_axis(lambda v: np.convolve(np.pad(v, r, mode="wrap"), k, "valid"),
                                axis, g)
    return (g - g.mean()) / (g.std() + 1e-300)


def generate_masked(nx, ny, nz, active_fraction=0.42, sigma=(2.0, 6.0, 4.0),
                    seed=2309, block_size=3, tx=1.0, ty=1.0, tz=0.5,
                    diagonal_boost=1.0) -> SystemBundle:
    """C2: NORNE-like irregular sparsity from a seeded inactive-cell mask.

    The mask thresholds a smoothed Gaussian field (array order [iz, iy, ix])
    at its ``1 - active_fraction`` quantile; active cells keep natural order.
    """
    rng = np.random.default_rng(seed)
    field = _smooth_field((nz, ny, nx), sigma, rng).reshape(-1)
    thr = np.quantile(field, 1.0 - active_fraction)
    active = field > thr
    new_id = np.cumsum(active) - 1
    faces = _faces(nx, ny, nz, active)
    lo = np.concatenate([new_id[f[0]] for f in faces])
    hi = np.concatenate([new_id[f[1]] for f in faces])
    t = np.concatenate([np.full(f[0].size, tv) for f, tv in zip(faces, (tx, ty, tz))])
    n = int(active.sum())
    rp, ci, blk = _assemble(n, lo, hi, t, block_size, diagonal_boost, rng)
    rhs = rng.uniform(-1.0, 1.0, size=n * block_size)
    return _bundle(rp, ci, blk, rhs, block_size, f"masked-{nx}x{ny}x{nz}-{n}", (nx, ny, nz))


def generate_heterogeneous(nx, ny, nz, sigma_k=2.5, corr=(2.0, 2.0, 1.0), seed=7,
                           block_size=3, tx=1.0, ty=1.0, tz=0.1,
                           diagonal_boost=1e-4) -> SystemBundle:
    """C3: heterogeneous permeability k = exp(sigma_k * g); each face's
    transmissibility is the harmonic mean of its two cells' k times the
    direction factor (tz << tx).  Small boost makes it ill-conditioned."""
    rng = np.random.default_rng(seed)
    g = _smooth_field((nz, ny, nx), corr[::-1], rng).reshape(-1)
    k = np.exp(sigma_k * g)
    faces = _faces(nx, ny, nz)
    lo = np.concatenate([f[0] for f in faces])
    hi = np.concatenate([f[1] for f in faces])
    tdir = np.concatenate([np.full(f[0].size, tv) for f, tv in zip(faces, (tx, ty, tz))])
    t = tdir * 2.0 * k[lo] * k[hi] / (k[lo] + k[hi])
    n = nx * ny * nz
    rp, ci, blk = _assemble(n, lo, hi, t, block_size, diagonal_boost, rng)
    rhs = rng.uniform(-1.0, 1.0, size=n * block_size)
    return _bundle(rp, ci, blk, rhs, block_size, f"hetero-{nx}x{ny}x{nz}", (nx, ny, nz))
