"""Parallelism extraction on the GPU: level scheduling, colouring, reordering.

Same API and results as ``bs/analysis.py`` (integer outputs bit-exact):
``level_schedule`` and ``graph_color`` run as sync-free device wavefronts
(csrc/analysis.cu), the stable group order comes from a device radix sort,
and ``apply_permutation`` permutes and re-sorts block rows on the device.
A :class:`ParallelPlan` keeps its arrays on the GPU and materialises the
reference's numpy views only when they are read.
"""

from __future__ import annotations

import enum

import numpy as np
import torch

from . import _device as D
from .blockcore import BlockMatrix, BlockVector, Layout, SparsityPattern, convert_layout
from .errors import ShapeError


class Strategy(enum.Enum):
    SEQUENTIAL = "sequential"
    LEVEL_SCHEDULING = "level-scheduling"
    GRAPH_COLORING = "graph-coloring"


class ParallelPlan:
    """Group per row + the stable permutation making groups contiguous
    (bs/analysis.py:28-58).  ``permutation[old] -> new``,
    ``inverse_permutation[new] -> old``, group g = rows
    ``[group_offsets[g], group_offsets[g+1])`` of the permuted order."""

    def __init__(self, strategy: Strategy, row_group=None, group_offsets=None,
                 permutation=None, inverse_permutation=None, *, _dev=None,
                 _ngroups=None, _identity=None, _independent=False):
        self.strategy = strategy
        # True when every group is an independent set of the pattern it was
        # built from (level / colour / sequential plans made here)
        self.independent_groups = _independent
        self._host = {}
        self._dev = _dev or {}
        for name, arr in (("row_group", row_group), ("group_offsets", group_offsets),
                          ("permutation", permutation),
                          ("inverse_permutation", inverse_permutation)):
            if arr is not None:
                self._host[name] = np.asarray(arr, dtype=np.int64)
        if _ngroups is None:
            _ngroups = len(self._host["group_offsets"]) - 1
        self._ngroups = int(_ngroups)
        self._n = (int(self._dev["row_group"].numel()) if "row_group" in self._dev
                   and "row_group" not in self._host else len(self._host["row_group"]))
        self._identity = _identity
        self._smap = None

    # -- reference attributes (numpy, int64) --------------------------------
    def _get(self, name):
        if name not in self._host:
            self._host[name] = self._dev[name][: self._len(name)].cpu().numpy().astype(np.int64)
        return self._host[name]

    def _len(self, name):
        return self._ngroups + 1 if name == "group_offsets" else self._n

    row_group = property(lambda self: self._get("row_group"))
    group_offsets = property(lambda self: self._get("group_offsets"))
    permutation = property(lambda self: self._get("permutation"))
    inverse_permutation = property(lambda self: self._get("inverse_permutation"))

    @property
    def num_rows(self) -> int:
        return self._n

    @property
    def group_count(self) -> int:
        return self._ngroups

    @property
    def largest_group(self) -> int:
        return int(np.diff(self.group_offsets).max()) if self.group_count else 0

    def rows_in_group(self, g: int) -> np.ndarray:
        off = self.group_offsets
        return self.inverse_permutation[off[g]:off[g + 1]]

    def __repr__(self):
        return f"ParallelPlan({self.strategy.value}, rows={self._n}, groups={self._ngroups})"

    # -- device side ----------------------------------------------------------
    def device(self, name: str) -> torch.Tensor:
        """int32 device copy of one of the plan arrays."""
        if name not in self._dev:
            dev = D.require_cuda()
            self._dev[name] = D.i32(self._host[name], dev)
        return self._dev[name]

    @property
    def is_identity(self) -> bool:
        if self._identity is None:
            if self.strategy is Strategy.SEQUENTIAL and "permutation" not in self._host:
                self._identity = True
            else:
                self._identity = bool(np.array_equal(self.permutation, np.arange(self._n)))
        return self._identity

    def slice_map(self):
        """Group-aligned SELL slices (rows of a slice are one group)."""
        if self._smap is None:
            self._smap = D.SliceMap.grouped(self.device("group_offsets"), self._ngroups)
        return self._smap


def _device_plan(strategy: Strategy, g: torch.Tensor, n: int, ngroups: int) -> ParallelPlan:
    perm, iperm, off = D.plan_arrays(g, n, ngroups)
    # one group keeps the stable order => identity; otherwise treat the plan as
    # a permutation (an identity that is permuted anyway costs a copy, not a
    # wrong answer) and spare the device->host check
    return ParallelPlan(strategy, _dev={"row_group": g, "permutation": perm,
                                        "inverse_permutation": iperm, "group_offsets": off},
                        _ngroups=ngroups, _independent=True, _identity=(ngroups <= 1))


def sequential_plan(num_rows: int) -> ParallelPlan:
    """One row per group in natural order (bs/analysis.py:74-76)."""
    idx = np.arange(num_rows, dtype=np.int64)
    return ParallelPlan(Strategy.SEQUENTIAL, idx, np.arange(num_rows + 1, dtype=np.int64),
                        idx, idx.copy(), _identity=True, _independent=True)


def level_schedule(p: SparsityPattern) -> ParallelPlan:
    """Levels of the strict-lower dependency DAG (bs/analysis.py:85-100)."""
    dp = D.DevPattern.upload(p)
    if dp.n == 0:
        return ParallelPlan(Strategy.LEVEL_SCHEDULING, np.zeros(0), [0], np.zeros(0),
                            np.zeros(0))
    g, ng = D.groups(dp, "level")
    return _device_plan(Strategy.LEVEL_SCHEDULING, g, dp.n, ng)


def graph_color(p: SparsityPattern) -> ParallelPlan:
    """Greedy first-fit colouring, ascending rows (bs/analysis.py:122-145)."""
    dp = D.DevPattern.upload(p)
    if dp.n == 0:
        return ParallelPlan(Strategy.GRAPH_COLORING, np.zeros(0), [0], np.zeros(0), np.zeros(0))
    g, ng = D.groups(dp, "color")
    return _device_plan(Strategy.GRAPH_COLORING, g, dp.n, ng)


def _check_plan(plan: ParallelPlan, num_rows: int):
    if plan.num_rows != num_rows:
        raise ShapeError("plan was built for a different number of rows")


def apply_permutation_vec(v: BlockVector, plan: ParallelPlan, inverse: bool = False) -> BlockVector:
    """v'[permutation[i]] = v[i] (bs/analysis.py:153-159), on the device."""
    _check_plan(plan, v.num_blocks)
    if v.num_blocks == 0:
        return BlockVector(v.data.copy(), v.block_size)
    dev = D.require_cuda()
    src = plan.device("permutation" if inverse else "inverse_permutation")
    out = D.gather_rows(D.f64(v.data, dev), src, v.num_blocks, v.block_size)
    return BlockVector(out.cpu().numpy(), v.block_size)


def permute_device(bsr: "D.DevBSR", plan: ParallelPlan, inverse: bool = False, want_src=False):
    cmap = plan.device("inverse_permutation" if inverse else "permutation")
    take = plan.device("permutation" if inverse else "inverse_permutation")
    return D.permute(bsr, cmap, take, want_src)


def dev_to_matrix(m: "D.DevBSR", layout: Layout = Layout.BLOCK_ROW_MAJOR) -> BlockMatrix:
    rp, ci = m.pat.host()
    bb = m.b * m.b
    vals = m.vals[: m.pat.nnz * bb].cpu().numpy()
    out = BlockMatrix(SparsityPattern(m.pat.n, rp, ci), m.b, vals, Layout.BLOCK_ROW_MAJOR)
    return out if layout is Layout.BLOCK_ROW_MAJOR else convert_layout(out, layout)


def apply_permutation(m: BlockMatrix, plan: ParallelPlan, inverse: bool = False) -> BlockMatrix:
    """Symmetric row/column reorder with re-sorted rows (bs/analysis.py:162-197)."""
    _check_plan(plan, m.num_block_rows)
    if m.num_block_rows == 0:
        return m.copy()
    out = permute_device(D.DevBSR.upload(m), plan, inverse)
    return dev_to_matrix(out, m.layout)
