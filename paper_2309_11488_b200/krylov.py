"""Right-preconditioned BiCGStab on the GPU (drop-in for bs/krylov.py).

``bicgstab(MatrixOperator(A), decompose(A, plan), b)`` runs entirely on the
device through the native driver ``b2s_bicgstab`` (csrc/krylov.cu): the
Krylov vectors live in plan order next to the plan-ordered operator and the
ILU factors, one iteration is one CUDA-graph replay, and the host only reads
a pinned completion word.  The reference's semantics are kept exactly:
half-step counting, the 1e-60 breakdown floor, the order of the exit tests,
the true-residual ``final_norm`` and the x0 return on non-finite x.

Other operator / preconditioner combinations the reference accepts (any
callable preconditioner, duck-typed operators) run a host-driven loop over
device vectors with the same control flow.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _device as D
from ._lib import BicgArgs, BicgResult, check
from .blockcore import BlockMatrix, BlockVector, DeviceOperator
from .errors import ShapeError
from .ilu0 import Ilu0Factorization

REDUCTION_CHUNK = 64          # bs/krylov.py:24
DEFAULT_REDUCTION = 0.01
DEFAULT_MAX_ITERATIONS = 200
_BREAKDOWN_FLOOR = 1e-60
_REASONS = {2: "breakdown", 3: "numerical", 4: "budget"}


# ---------------------------------------------------------------------------
# reductions

def dot_partials(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-chunk partial sums of a*b over consecutive 64-element chunks
    (bs/krylov.py:30-36), computed on the device in numpy's exact order."""
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    if a.size == 0:
        return np.zeros(0)
    dev = D.require_cuda()
    return D.dot_chunked(D.f64(a, dev), D.f64(b, dev), a.size, partials=True).cpu().numpy()


def dot_arrays(a: np.ndarray, b: np.ndarray) -> float:
    """Chunk partials accumulated strictly left to right (bs/krylov.py:39-44):
    bit-identical to the reference (csrc/refdot.cu)."""
    a = np.asarray(a, dtype=np.float64).reshape(-1)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    if a.size == 0:
        return 0.0
    dev = D.require_cuda()
    return float(D.dot_chunked(D.f64(a, dev), D.f64(b, dev), a.size).item())


def norm_array(a: np.ndarray) -> float:
    return float(np.sqrt(dot_arrays(a, a)))


_SIDE: dict = {}


def _side_stream(dev: torch.device) -> torch.cuda.Stream:
    s = _SIDE.get(dev.index)
    if s is None:
        s = _SIDE[dev.index] = torch.cuda.Stream(device=dev)
    return s


class RefNorm:
    """``||r0||`` in the reference's summation order (bs/krylov.py:176,
    norm_array), computed on a side stream while the Krylov loop runs: the
    reported ``initial_norm`` is then bit-identical to
    ``norm_array(b - A x0)``; the loop's own stopping target uses its
    fixed-order device reduction (within an ulp of it)."""

    def __init__(self, r0: torch.Tensor, m: int):
        side = _side_stream(r0.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self._sq = D.dot_chunked(r0, r0, m) if m else None
            self._ev = torch.cuda.Event()
            self._ev.record(side)
        r0.record_stream(side)

    def value(self) -> float:
        self._ev.synchronize()
        return 0.0 if self._sq is None else float(np.sqrt(float(self._sq.item())))

    def fetch_into(self, tail: "D.HostResult"):
        """Queue the squared norm's D2H on the current stream (after the side
        stream's event) into ``tail``; ``from_tail`` reads it after wait()."""
        if self._sq is None:
            self._k = None
            return
        torch.cuda.current_stream().wait_event(self._ev)
        self._k = tail.fetch(self._sq.reshape(1))

    def from_tail(self, tail: "D.HostResult") -> float:
        if self._k is None:
            return 0.0
        return float(np.sqrt(float(tail.value(self._k)[0])))


def dot(a: BlockVector, b: BlockVector) -> float:
    """Deterministic chunked inner product of two block vectors (the
    reference's order, bit for bit)."""
    if a.data.size != b.data.size:
        raise ShapeError("vectors have different lengths")
    return dot_arrays(a.data, b.data)


def norm(a: BlockVector) -> float:
    return float(np.sqrt(dot(a, a)))


# ---------------------------------------------------------------------------
# operators and reports

class MatrixOperator:
    """Plain blocked SpMV operator (bs/krylov.py:63-81).

    The reference reads ``matrix.values`` at every apply.  Here the device copy
    is taken at the start of every public call (``apply_array``/``apply``,
    ``bicgstab``), so in-place changes to the host arrays between calls are
    always seen; inside one call the host arrays are read once."""

    def __init__(self, a: BlockMatrix):
        self.matrix = a.as_block_row_major()
        self._dev = None

    @property
    def block_size(self) -> int:
        return self.matrix.block_size

    @property
    def num_blocks(self) -> int:
        return self.matrix.num_block_rows

    def device(self, refresh: bool = False) -> DeviceOperator:
        if self._dev is None or refresh:
            self._dev = DeviceOperator(self.matrix)
        return self._dev

    def prepare(self):
        """Device copies of the current host arrays (start of a public call)."""
        self.device(refresh=True)

    def apply_device(self, x: torch.Tensor, y: torch.Tensor):
        self.device().apply(x, y)

    def apply_array(self, x: np.ndarray) -> np.ndarray:
        self.prepare()
        op = self.device()
        dev = op.bsr.pat.rp.device
        y = D.empty_f64(op.n * op.b, dev)
        self.apply_device(D.f64(x, dev), y)
        return y[: op.n * op.b].cpu().numpy()

    def apply(self, x: BlockVector) -> BlockVector:
        return BlockVector(self.apply_array(x.data), self.block_size)


class WellAugmentedOperator(MatrixOperator):
    """SpMV followed by every well's -C^T D^-1 B x (bs/krylov.py:84-94), both on
    the device (csrc/spmv.cu, csrc/wells.cu).  Like the reference
    (wells.apply_contributions_array), a COUPLED or empty set adds nothing:
    its wells are already folded into the matrix."""

    def __init__(self, a: BlockMatrix, wells):
        super().__init__(a)
        self.wells = wells

    def _separate(self) -> bool:
        from .wells import WellMode
        return self.wells.mode is not WellMode.COUPLED and not self.wells.is_empty

    def apply_device(self, x: torch.Tensor, y: torch.Tensor):
        self.device().apply(x, y)
        if self._separate():
            self.wells.device(self.block_size, self.num_blocks).apply(x, y)


@dataclass(frozen=True)
class StoppingCriteria:
    """Relative residual reduction and iteration budget (bs/krylov.py:97-108)."""

    relative_reduction: float = DEFAULT_REDUCTION
    max_iterations: int = DEFAULT_MAX_ITERATIONS

    def __post_init__(self):
        if not 0.0 < self.relative_reduction < 1.0:
            raise ValueError("relative_reduction must lie in (0, 1)")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be >= 1")


@dataclass
class SolveReport:
    """Outcome of one solve (bs/krylov.py:111-129); iterations in half steps."""

    converged: bool
    iterations: float
    initial_norm: float
    final_norm: float
    elapsed: float
    group_count: int
    fallback_used: bool = False
    failure_reason: str | None = None
    setup_elapsed: float = 0.0
    # device-side accounting (not in the reference): graph replays and kernels
    gpu_launches: int = 0
    # B2S_TRACE=1: {phase: (host_ms, gpu_ms)} (paper_2309_11488_b200/trace.py)
    phases: dict | None = None


# ---------------------------------------------------------------------------
# the native driver

@dataclass
class DeviceKrylov:
    """Everything ``b2s_bicgstab`` needs, resident in plan order."""

    n: int
    b: int
    smap: "D.SliceMap"
    a: "D.Sell"
    fact: Ilu0Factorization | None
    work: torch.Tensor
    fuse: bool = False   # 2-colour fused backward + SpMV passes (csrc/fused.cu)
    wells: object = None   # DeviceWells in this solver's row order (separate wells)
    wtabs: tuple = ()      # its WellFix tables (slice, lane, corr)

    @classmethod
    def build(cls, matrix: BlockMatrix, fact: Ilu0Factorization | None,
              a_bsr: "D.DevBSR" = None, same_values: bool = False,
              wells=None) -> "DeviceKrylov":
        """``same_values``: the caller guarantees ``matrix``'s host values are
        the ones ``fact`` was computed from (one solve_with_fallback call), so
        the factorisation's device copy of them can serve as the operator.
        Otherwise (public bicgstab) the operator is uploaded afresh.
        ``wells``: a WellSet applied separately (WellAugmentedOperator): its
        terms run inside the device loop, in the plan's row order."""
        n, b = matrix.num_block_rows, matrix.block_size
        fuse_env = os.environ.get("B2S_FUSE", "1") != "0"
        sell = None
        if fact is not None:
            smap = fact.smap
            reuse = same_values and fact._source is matrix
            shell = fact._op_shell if reuse else None
            if a_bsr is None and fact.a_sell is not None and reuse:
                sell = fact.a_sell   # 2-colour factorisation: the operator layout exists
            elif a_bsr is None and fact._a_src is not None and reuse:
                ppat, src, inp = fact._a_src   # filled from the unpermuted input values
                if shell is not None:   # sized in the pattern phase: values only now
                    sell = shell
                    sell.fill_from(smap, D.DevBSR(ppat, b, inp.vals), 0, src)
                else:
                    sell = D.Sell.build(smap, D.DevBSR(ppat, b, inp.vals), 0, src=src)
            elif a_bsr is None and shell is not None and fact._a_perm is not None:
                sell = shell        # identity plan: the input is the operator
                sell.fill_from(smap, fact._a_perm, 0)
            elif a_bsr is None:
                a_bsr = (fact._a_perm if reuse and fact._a_perm is not None
                         else _plan_order(D.DevBSR.upload(matrix), fact))
            dev = fact.dtiles.device
        else:
            a_bsr = a_bsr or D.DevBSR.upload(matrix)
            dev = a_bsr.pat.rp.device
            smap = D.SliceMap.plain(n, dev)
        if sell is None:
            sell = D.Sell.build(smap, a_bsr, 0)
        nbytes = int(D.lib().b2s_bicgstab_workspace_bytes(n, b, D.NPARTS))
        work = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=dev)
        fuse = False
        dw, wtabs = None, ()
        if wells is not None and not wells.is_empty:
            # the input-order packing is cached on the WellSet (while its
            # arrays are unchanged); the plan-order view is built on the device
            dw0 = wells.device(b, n)
            if fact is not None and not fact._identity_perm:
                perm = fact.plan.device("permutation")   # old row -> plan row
            else:
                perm = torch.arange(n, dtype=torch.int32, device=dev)
            dw = dw0.in_plan_order(perm, smap)
            wtabs = dw.tables
        if sell is not None and fact is not None and sell is fact.a_sell:
            # U's colour-0 rows are this very layout (factor2c.cu): fusable by construction
            fuse = fact.phased and fuse_env
        elif (fact is not None and fact.phased and not fact.tiles and
                len(smap.gslice_host) == 3 and fuse_env):
            ok = C.c_int32(0)
            up = fact.upper
            check(D.lib().b2s_fuse_check(int(smap.gslice_host[1]), b, D.ptr(smap.row0),
                                         D.ptr(smap.nrows), D.ptr(sell.sp), D.ptr(sell.cols),
                                         D.ptr(sell.vals), D.ptr(up.sp), D.ptr(up.cols),
                                         D.ptr(up.vals), C.byref(ok), D.stream()), "fuse_check")
            fuse = bool(ok.value)
        return cls(n, b, smap, sell, fact, work, fuse, dw, wtabs)

    def solve(self, rhs: torch.Tensor, x: torch.Tensor, stop: StoppingCriteria,
              check_lag: int = 2, mesh=None, x0_zero: bool = False) -> BicgResult:
        """Solve in place on plan-order device vectors (x: x0 in, x out).
        ``mesh``: a ``_lib.Mesh`` for one shard of a partitioned solve (x then
        carries the ghost rows after the owned ones; distributed.py)."""
        f = self.fact
        args = BicgArgs()
        args.n, args.b, args.nparts = self.n, self.b, D.NPARTS
        args.precond = 1 if f is not None else 0
        args.kc = f.kc if f is not None else 2
        args.maxit = stop.max_iterations
        args.check_lag = check_lag
        args.refill_y = 1 if (f is not None and not self.fuse and not f.gw and
                              f.upper.stale) else 0
        args.sweep_flags = f.sweep_flags if f is not None else 0
        args.tol = stop.relative_reduction
        s = self.smap
        args.nslices, args.row0, args.nrows = s.nslices, D.ptr(s.row0), D.ptr(s.nrows)
        args.a_sp, args.a_cols, args.a_vals = D.ptr(self.a.sp), D.ptr(self.a.cols), D.ptr(self.a.vals)
        if f is not None:
            if not f.gw:   # (the wavefront sweeps read their own packed records)
                args.l_sp, args.l_cols, args.l_vals = (D.ptr(f.lower.sp), D.ptr(f.lower.cols),
                                                       D.ptr(f.lower.vals))
            if not self.fuse and not f.gw:   # (the fused passes read U's rows from the operator)
                args.u_sp, args.u_cols, args.u_vals = (D.ptr(f.upper.sp), D.ptr(f.upper.cols),
                                                       D.ptr(f.upper.vals))
            args.dinv_tiles = D.ptr(f.dtiles)
            args.tiles = f.tiles
            args.gw = f.gw
            if f.phased and not f.tiles:
                args.ngroups = len(s.gslice_host) - 1
                args.goff1 = s.goff1
                args.gslice_host = s.gslice_host.ctypes.data
                args.fuse = 1 if self.fuse else 0
        args.rhs, args.x, args.work = D.ptr(rhs), D.ptr(x), D.ptr(self.work)
        args.stream = D.stream()
        if mesh is not None:
            args.mesh = C.addressof(mesh)
        args.x0_zero = 1 if x0_zero else 0   # caller guarantees x == 0 on entry
        if self.wells is not None and self.wells.nwells:
            args.wells = C.addressof(self.wells._args)
            sl, ln, corr = self.wtabs
            args.well_slice, args.well_lane, args.well_corr = D.ptr(sl), D.ptr(ln), D.ptr(corr)
            args.well_scratch = D.ptr(self.wells.scratch)
        res = BicgResult()
        check(D.lib().b2s_bicgstab(C.byref(args), C.byref(res)), "bicgstab")
        return res


def _plan_order(bsr: "D.DevBSR", fact: Ilu0Factorization) -> "D.DevBSR":
    from .analysis import permute_device
    return bsr if fact._identity_perm else permute_device(bsr, fact.plan)


def _as_precond(precond) -> Callable[[np.ndarray], np.ndarray]:
    if precond is None:
        return lambda r: r
    if isinstance(precond, Ilu0Factorization):
        return precond.apply_array
    return precond


def bicgstab(op, precond, b: BlockVector, x0: BlockVector | None = None,
             stop: StoppingCriteria | None = None) -> tuple[BlockVector, SolveReport]:
    """Solve op(x) = b with right-preconditioned BiCGStab (bs/krylov.py:140-244)."""
    if stop is None:
        stop = StoppingCriteria()
    if b.block_size != op.block_size or b.num_blocks != op.num_blocks:
        raise ShapeError("right-hand side does not match the operator")
    x0_given = x0 is not None
    if x0 is None:
        x0 = BlockVector.zeros(op.num_blocks, op.block_size)
    elif x0.block_size != b.block_size or x0.num_blocks != b.num_blocks:
        raise ShapeError("initial guess does not match the right-hand side")
    native = (type(op) in (MatrixOperator, WellAugmentedOperator) and
              (precond is None or isinstance(precond, Ilu0Factorization)) and
              op.num_blocks > 0)
    # WellAugmentedOperator and other operators/preconditioners: host-driven
    # loop over device vectors (device operators stay on the device)
    if native:
        return _bicgstab_native(op, precond, b, x0, stop, x0_zero=x0_given is False)
    return _bicgstab_generic(op, precond, b, x0, stop)


def _bicgstab_native(op: MatrixOperator, fact, b: BlockVector, x0: BlockVector,
                     stop: StoppingCriteria, krylov: DeviceKrylov | None = None,
                     x0_zero: bool = False):
    t0 = time.perf_counter()
    wells = op.wells if isinstance(op, WellAugmentedOperator) and op._separate() else None
    kr = krylov or DeviceKrylov.build(op.matrix, fact, wells=wells)
    n, bs = kr.n, kr.b
    dev = kr.work.device
    bd, xd = D.f64(b.data, dev), D.f64(x0.data, dev)
    if x0_zero:
        r0 = bd
    else:   # input-order residual through the public operator (bs/krylov.py:175)
        op.prepare()
        y = D.empty_f64(n * bs, dev)
        op.apply_device(xd, y)
        r0 = bd - y[: n * bs]
    norm0 = RefNorm(r0, n * bs)
    perm = fact is not None and not fact._identity_perm
    if perm:
        iperm = fact.plan.device("inverse_permutation")
        bd, xd = D.gather_rows(bd, iperm, n, bs), D.gather_rows(xd, iperm, n, bs)
    res = kr.solve(bd, xd, stop, x0_zero=x0_zero)
    if perm:
        xd = D.gather_rows(xd, fact.plan.device("permutation"), n, bs)
    x = D.to_host(xd, n * bs)
    groups = fact.plan.group_count if fact is not None else 0
    rep = SolveReport(bool(res.converged), float(res.iterations), norm0.value(),
                      float(res.final_norm), time.perf_counter() - t0, groups,
                      failure_reason=None if res.converged else _REASONS.get(res.reason, "budget"),
                      gpu_launches=int(res.graph_launches) * int(res.kernels_per_iteration))
    if not res.converged and res.reason == 3 and res.iterations == 0.0 and \
            not np.isfinite(res.initial_norm):
        x = x0.data.copy()
    return BlockVector(x, bs), rep


def _bicgstab_generic(op, precond, b: BlockVector, x0: BlockVector, stop: StoppingCriteria):
    """Host-driven loop for duck-typed operators / callable preconditioners;
    vectors stay on the device, reductions use the device dot kernel."""
    apply_m = _as_precond(precond)
    groups = precond.plan.group_count if isinstance(precond, Ilu0Factorization) else 0
    t0 = time.perf_counter()
    dev = D.require_cuda()
    m = b.data.size

    if hasattr(op, "prepare"):
        op.prepare()
    if hasattr(op, "apply_device"):
        def A(v):   # device operator (SpMV [+ wells]): no host round trip
            y = torch.empty_like(v)
            op.apply_device(v, y)
            return y
    else:
        def A(v):   # duck-typed operator: through its array API
            return D.f64(op.apply_array(v.cpu().numpy()), dev)

    if isinstance(precond, Ilu0Factorization) and m:
        f = precond

        def M(v):   # device ILU0 application in plan order
            if f._identity_perm:
                return f.apply_device(v)[:m]
            vp = D.gather_rows(v, f.plan.device("inverse_permutation"), f.num_block_rows,
                               f.block_size)
            z = f.apply_device(vp)
            return D.gather_rows(z, f.plan.device("permutation"), f.num_block_rows,
                                 f.block_size)[:m]
    else:
        def M(v):
            return D.f64(apply_m(v.cpu().numpy()), dev)

    def dt(u, v):   # the reference's chunk-64 order, bit for bit (csrc/refdot.cu)
        return float(D.dot_chunked(u, v, m).item()) if m else 0.0

    def nrm(v):
        return float(np.sqrt(dt(v, v)))

    x = D.f64(x0.data, dev) if m else torch.zeros(0, dtype=torch.float64, device=dev)
    bd = D.f64(b.data, dev) if m else x.clone()
    r = bd - A(x) if m else x.clone()
    norm0 = nrm(r)
    target = stop.relative_reduction * norm0

    def report(conv, its, final, reason=None):
        return SolveReport(conv, its, norm0, final, time.perf_counter() - t0, groups,
                           failure_reason=reason)

    if not np.isfinite(norm0):
        return BlockVector(x0.data.copy(), b.block_size), report(False, 0.0, norm0, "numerical")
    if norm0 <= target or norm0 == 0.0:
        return BlockVector(x.cpu().numpy(), b.block_size), report(True, 0.0, norm0)
    rhat = r.clone()
    rho_prev = alpha = omega = 1.0
    v = torch.zeros_like(r)
    p = torch.zeros_like(r)
    its = 0.0
    reason = "budget"
    for k in range(stop.max_iterations):
        rho = dt(rhat, r)
        if abs(rho) < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        p = r.clone() if k == 0 else r + ((rho / rho_prev) * (alpha / omega)) * (p - omega * v)
        phat = M(p)
        v = A(phat)
        gamma = dt(rhat, v)
        if abs(gamma) < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        alpha = rho / gamma
        s = r - alpha * v
        x = x + alpha * phat
        its += 0.5
        ns = nrm(s)
        if not np.isfinite(ns):
            reason = "numerical"
            break
        if ns <= target:
            return BlockVector(x.cpu().numpy(), b.block_size), report(True, its, ns)
        shat = M(s)
        t = A(shat)
        tt = dt(t, t)
        if tt < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        omega = dt(t, s) / tt
        if abs(omega) < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        x = x + omega * shat
        r = s - omega * t
        its += 0.5
        nr = nrm(r)
        if not np.isfinite(nr):
            reason = "numerical"
            break
        if nr <= target:
            return BlockVector(x.cpu().numpy(), b.block_size), report(True, its, nr)
        rho_prev = rho
    final = nrm(bd - A(x))
    xh = x.cpu().numpy()
    out = xh if np.all(np.isfinite(xh)) else x0.data.copy()
    return BlockVector(out, b.block_size), report(False, its, final, reason)
