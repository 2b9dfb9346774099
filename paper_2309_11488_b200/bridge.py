"""Backend registry, solve orchestration and the sequential fallback
(drop-in for bs/bridge.py).

``solve_with_fallback`` keeps the reference's contract: build the operator,
optionally Jacobi-relax the preconditioner matrix, extract parallelism per
backend, factor, run BiCGStab, and on failure (not converged or singular
pivot) rerun with the sequential ILU0 of the full matrix and at least the
default budget; raise ``SolveFailed`` when that fails too.

B200 specifics: the matrix crosses to the GPU once per call; analysis,
permutation, factorisation, the Krylov loop and the fallback all run on it,
and only the solution vector comes back.  :class:`DeviceSolver` exposes the
same pipeline for device-resident inputs (benchmarks, repeated solves).
"""

from __future__ import annotations

import enum
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import trace
from .analysis import (ParallelPlan, Strategy, _device_plan, sequential_plan)
from .blockcore import BlockMatrix, BlockVector
from .errors import SingularPivot, SolveFailed
from .ilu0 import Ilu0Factorization, factor_device, prepare_general, prepare_two_colour
from .krylov import (DEFAULT_MAX_ITERATIONS, DeviceKrylov, RefNorm, SolveReport,
                     StoppingCriteria, _REASONS)
from .wells import WellMode, WellSet, fold_into_matrix


class Backend(enum.Enum):
    """Same members as bs/bridge.py:26-37 (tests iterate over the enum and
    reject unknown names such as "gpu"); every member runs on the B200."""

    REFERENCE_SEQUENTIAL = "reference"
    LEVEL_SCHEDULED = "level"
    GRAPH_COLORED = "color"

    @classmethod
    def from_name(cls, name: str) -> "Backend":
        for member in cls:
            if member.value == name:
                return member
        raise ValueError(f"unknown backend {name!r}; choose from {[m.value for m in cls]}")


@dataclass(frozen=True)
class SolverConfig:
    """bs/bridge.py:40-55."""

    backend: Backend = Backend.LEVEL_SCHEDULED
    jacobi_partitions: int = 0
    well_mode: WellMode = WellMode.SEPARATE
    stop: StoppingCriteria = field(default_factory=StoppingCriteria)

    def __post_init__(self):
        if self.jacobi_partitions < 0:
            raise ValueError("jacobi_partitions must be >= 0")


def plan_device(backend: Backend, pat: "D.DevPattern") -> ParallelPlan:
    """_plan_for (bs/bridge.py:58-63) on an uploaded pattern."""
    if backend is Backend.LEVEL_SCHEDULED:
        g, ng = D.groups(pat, "level")
        return _device_plan(Strategy.LEVEL_SCHEDULING, g, pat.n, ng)
    if backend is Backend.GRAPH_COLORED:
        g, ng = D.groups(pat, "color")
        return _device_plan(Strategy.GRAPH_COLORING, g, pat.n, ng)
    return sequential_plan(pat.n)


def _failed_report(reason: str) -> SolveReport:
    return SolveReport(False, 0.0, float("nan"), float("nan"), 0.0, 0, failure_reason=reason)


class DeviceSolver:
    """The whole reference pipeline on device-resident data.

    ``setup()`` = analysis + permutation + factorisation + operator layout;
    ``solve(rhs, x)`` = BiCGStab on plan-ordered device vectors.  Inputs and
    outputs are torch CUDA tensors in the matrix's own row order.
    """

    def __init__(self, a: BlockMatrix, bsr: "D.DevBSR", cfg: SolverConfig,
                 precond_bsr: "D.DevBSR" = None, precond_matrix: BlockMatrix = None,
                 wells: WellSet | None = None):
        self.a = a
        self.wells = wells if wells is not None and not wells.is_empty else None
        self.bsr = bsr
        self.cfg = cfg
        self.pre_bsr = precond_bsr or bsr
        self.pre_matrix = precond_matrix or a
        self.fact: Ilu0Factorization | None = None
        self.krylov: DeviceKrylov | None = None
        self.plan: ParallelPlan | None = None

    def setup(self, backend: Backend | None = None, two_colour: bool = True,
              defer: bool = True, pattern_phase=None):
        """``defer``: the factorisation's pivot check is read after the solve
        (solve() raises SingularPivot then); False raises it here.
        ``pattern_phase``: (plan, prep, prep_general) kept by a SolveSession
        from an earlier solve on the same pattern."""
        backend = backend or self.cfg.backend
        self._backend = backend
        with trace.phase("analysis"):
            if pattern_phase is not None:
                self.plan, prep, prep_g = pattern_phase
            else:
                self.plan = plan_device(backend, self.pre_bsr.pat)
                # the pattern-only part of the factorisation, also before the values
                prep = (prepare_two_colour(self.pre_matrix, self.plan, self.pre_bsr.pat)
                        if two_colour else None)
                prep_g = (prepare_general(self.pre_matrix, self.plan, self.pre_bsr.pat)
                          if prep is None else None)
        with trace.phase("wait_values"):
            self.pre_bsr.wait_values()   # values may still be in flight (overlapped upload)
            self.bsr.wait_values()
        with trace.phase("factor"):
            # a 2-colour factorisation's pivot / structure check is read after
            # the solve (solve() below): the host builds and launches the loop
            # while the device factorises
            self.fact = factor_device(self.pre_matrix, self.plan, self.pre_bsr, prep, defer=defer,
                                      two_colour=two_colour, prep_general=prep_g)
        w = self.wells
        if self.pre_bsr is self.bsr and self.fact.a_sell is not None:
            # 2-colour factorisation: the operator's SELL layout already exists
            self.krylov = DeviceKrylov.build(self.a, self.fact, same_values=True, wells=w)
            return self
        a_perm = self.fact._a_perm if self.pre_bsr is self.bsr else None
        if a_perm is None and self.pre_bsr is self.bsr and self.fact._a_src is not None:
            self.krylov = DeviceKrylov.build(self.a, self.fact, same_values=True,
                                             wells=w)   # from the input
            return self
        if a_perm is None:
            from .analysis import permute_device
            a_perm = (self.bsr if self.fact._identity_perm
                      else permute_device(self.bsr, self.plan))
        self.krylov = DeviceKrylov.build(self.a, self.fact, a_perm, wells=w)
        return self

    def solve(self, rhs: torch.Tensor, x: torch.Tensor, stop: StoppingCriteria,
              x0_zero: bool = False, on_done=None):
        """x (input order) holds x0 on entry and the solution on exit;
        ``x0_zero``: the caller guarantees x == 0 (no initial guess).
        A deferred factorisation check runs after the loop: SingularPivot is
        raised as decompose would have; a pattern that was not a 2-colour
        structure after all is refactorised on the general path and solved
        again from the same x0.  ``on_done()`` runs after each solve is
        queued and before the check reads the flags, so the caller's result
        reads join that one synchronisation."""
        pending = self.fact._deferred is not None
        x_in = x.clone() if pending and not x0_zero else None
        res = self._solve(rhs, x, stop, x0_zero)
        if on_done is not None:
            on_done()
        if pending and self.fact.check_deferred():
            self.setup(self._backend, two_colour=False, defer=False)
            if x_in is None:
                x.zero_()
            else:
                x.copy_(x_in)
            res = self._solve(rhs, x, stop, x0_zero)
            if on_done is not None:
                on_done()
        return res

    def _solve(self, rhs: torch.Tensor, x: torch.Tensor, stop: StoppingCriteria,
               x0_zero: bool = False):
        n, b = self.krylov.n, self.krylov.b
        f = self.fact
        if f._identity_perm:
            return self.krylov.solve(rhs, x, stop, x0_zero=x0_zero)
        iperm = f.plan.device("inverse_permutation")
        bp = D.gather_rows(rhs, iperm, n, b)
        xp = D.gather_rows(x, iperm, n, b)
        res = self.krylov.solve(bp, xp, stop, x0_zero=x0_zero)
        D.gather_rows(xp, f.plan.device("permutation"), n, b, out=x)
        return res


def _report(res, elapsed, groups, norm0: float | None = None) -> SolveReport:
    n0 = float(res.initial_norm) if norm0 is None else norm0
    return SolveReport(bool(res.converged), float(res.iterations), n0,
                       float(res.final_norm), elapsed, groups,
                       failure_reason=None if res.converged else _REASONS.get(res.reason, "budget"),
                       gpu_launches=int(res.graph_launches) * int(res.kernels_per_iteration))


class _Tail:
    """The end-of-solve event and the queued host reads (D.HostResult) of
    x and the reported initial norm."""

    def __init__(self, x: torch.Tensor, count: int, block_size: int, norm0: "RefNorm"):
        self.x, self.count, self.block_size, self.norm0 = x, count, block_size, norm0
        self.end = self.host = None

    def __call__(self):
        self.end = torch.cuda.Event(enable_timing=True)
        self.end.record()
        self.host = D.HostResult(self.x, self.count, self.block_size)
        self.norm0.fetch_into(self.host)

    def wait(self):
        self.host.wait()
        return self.end, self.host


def _sync():
    torch.cuda.current_stream().synchronize()


def _initial_residual(bsr: "D.DevBSR", rhs: torch.Tensor, x0d: torch.Tensor | None,
                      wells: WellSet | None = None):
    """b - op(x0) in input order (bs/krylov.py:175; op = A, or A minus the
    separately applied wells, as WellAugmentedOperator.apply_array computes
    it) for the reported initial norm; b itself when there is no initial guess."""
    if x0d is None:
        return rhs
    n, b = bsr.pat.n, bsr.b
    smap = D.SliceMap.plain(n, rhs.device)
    y = D.empty_f64(n * b, rhs.device)
    D.spmv(smap, D.Sell.build(smap, bsr, 0), b, x0d, y)
    if wells is not None and not wells.is_empty:
        wells.device(b, n).apply(x0d, y)
    return rhs - y[: n * b]


def solve_with_fallback(cfg: SolverConfig, a: BlockMatrix, b: BlockVector, wells=None,
                        x0: BlockVector | None = None) -> tuple[BlockVector, SolveReport]:
    """Configured backend first, sequential ILU0 fallback second
    (bs/bridge.py:71-136)."""
    from .errors import ShapeError
    if wells is None:
        wells = WellSet()
    t0 = time.perf_counter()
    sep = None
    if cfg.well_mode is WellMode.COUPLED and not wells.is_empty:
        a_sys = fold_into_matrix(a, wells)          # host assembly, as the reference
    else:
        a_sys = a.as_block_row_major()
        if not wells.is_empty:
            # the config governs the treatment, whatever the set was marked as;
            # the well terms run inside the device loop (WellAugmentedOperator)
            sep = WellSet(wells.standard, wells.multisegment, WellMode.SEPARATE)
    n, bs = a_sys.num_block_rows, a_sys.block_size
    if b.block_size != bs or b.num_blocks != n:
        raise ShapeError("right-hand side does not match the operator")
    if x0 is not None and (x0.block_size != bs or x0.num_blocks != n):
        raise ShapeError("initial guess does not match the right-hand side")
    if n == 0:
        rep = SolveReport(True, 0.0, 0.0, 0.0, 0.0, 0)
        return BlockVector(np.zeros(0) if x0 is None else x0.data.copy(), bs), rep
    dev = D.require_cuda()
    trace.start()
    with trace.phase("upload"):
        # the 72 B/block values (the bulk of the upload) travel while the
        # device analyses the pattern; the solve waits for them only at
        # factorisation
        bsr = D.DevBSR.upload(a_sys, overlap=cfg.jacobi_partitions == 0)
        # the vectors queue behind the values on the copy stream: the
        # analysis (pattern only) must not wait for them
        rhs = bsr.upload_after(b.data)
        x0d = (torch.zeros(n * bs, dtype=torch.float64, device=dev) if x0 is None
               else bsr.upload_after(x0.data))

    pre_bsr, pre_mat = bsr, a_sys
    primary = None
    norm0 = None
    x = None
    try:
        if cfg.jacobi_partitions > 0:
            from .jacobi import relax_on_device
            bsr.wait_values()
            pre_mat = relax_on_device(a_sys, bsr, cfg.jacobi_partitions)
            pre_bsr = pre_mat.bsr
        solver = DeviceSolver(a_sys, bsr, cfg, pre_bsr, pre_mat, wells=sep).setup()
        # the reported ||r0|| in the reference's order, beside the loop
        norm0 = RefNorm(_initial_residual(bsr, rhs, None if x0 is None else x0d, sep), n * bs)
        # no host synchronisation between setup and solve: the phases are
        # timed on the device (the host queues the loop while the device is
        # still factorising)
        e_setup = torch.cuda.Event(enable_timing=True)
        e_setup.record()
        xd = x0d.clone()
        with trace.phase("krylov"):
            # everything the host reads next (deferred factor flags, x, the
            # initial norm) queued, then one synchronisation
            queue = _Tail(xd, n * bs, bs, norm0)
            res = solver.solve(rhs, xd, cfg.stop, x0_zero=x0 is None, on_done=queue)
        e_end, tail = queue.wait()
        setup = (time.perf_counter() - t0) - e_setup.elapsed_time(e_end) / 1e3
        primary = _report(res, e_setup.elapsed_time(e_end) / 1e3, solver.plan.group_count,
                          norm0.from_tail(tail))
        primary.setup_elapsed = max(setup, 0.0)
        x = xd
    except SingularPivot as exc:
        primary = _failed_report(f"singular pivot in row {exc.row}")
        primary.setup_elapsed = time.perf_counter() - t0

    if primary.converged:
        with trace.phase("download"):
            out = tail.vector()
        primary.phases = trace.finish()
        return out, primary

    fb_t0 = time.perf_counter()
    fb_stop = StoppingCriteria(cfg.stop.relative_reduction,
                               max(cfg.stop.max_iterations, DEFAULT_MAX_ITERATIONS))
    fcfg = SolverConfig(Backend.REFERENCE_SEQUENTIAL, 0, cfg.well_mode, fb_stop)
    try:
        fb = DeviceSolver(a_sys, bsr, fcfg, wells=sep).setup(defer=False)
    except SingularPivot as exc:
        fb_report = _failed_report(f"singular pivot in row {exc.row}")
        fb_report.fallback_used = True
        raise SolveFailed(primary, fb_report)
    if norm0 is None:   # the primary failed before its loop: ||r0|| from here
        norm0 = RefNorm(_initial_residual(bsr, rhs, None if x0 is None else x0d, sep), n * bs)
    _sync()
    fb_setup = time.perf_counter() - fb_t0
    t2 = time.perf_counter()
    xd = x0d.clone()
    res = fb.solve(rhs, xd, fb_stop, x0_zero=x0 is None)
    _sync()
    report = _report(res, time.perf_counter() - t2, n,
                     norm0.value() if norm0 is not None else None)
    report.fallback_used = True
    report.setup_elapsed = primary.setup_elapsed + fb_setup
    report.elapsed += primary.elapsed
    if not report.converged:
        raise SolveFailed(primary, report)
    return D.to_host_vector(xd, n * bs, bs), report


class _PatternStandIn:
    """What the pattern-only setup reads of a BlockMatrix (n, b, pattern)."""

    def __init__(self, pattern, block_size: int):
        self.pattern = pattern
        self.num_block_rows = pattern.num_block_rows
        self.block_size = block_size

    def as_block_row_major(self):
        return self


class SolveSession:
    """Repeated solves on one sparsity pattern -- a simulator's Newton loop,
    where every linear system has the same structure and new values.

    The pattern phase of ``solve_with_fallback`` (index upload, plan,
    permutation, slice maps, layout sizes, symbolic factorisation, the
    wavefront packing pattern) runs once, at construction; each ``solve``
    uploads only the block values and the right-hand side and runs the value
    phase (factorisation, layout fill) and the Krylov loop.  Results, reports
    and exceptions are those of ``solve_with_fallback(cfg, a, b, wells, x0)``
    bit for bit: a primary failure (singular pivot, no convergence) and
    systems the session cannot serve (another pattern, COUPLED wells, which
    fold into the matrix) go through ``solve_with_fallback`` itself.  (The
    reference has no such object: it re-analyses every call; this is the
    device-side analogue of its ``refresh_values`` reuse for partitions,
    ``bs/jacobi.py:139-147``.)  A session holds device buffers for one
    system at a time: use one session per thread (independent sessions and
    ``solve_with_fallback`` calls may run concurrently)."""

    def __init__(self, cfg: SolverConfig, pattern, block_size: int = 3):
        from .blockcore import SparsityPattern
        if not isinstance(pattern, SparsityPattern):
            raise TypeError("SolveSession needs a SparsityPattern")
        self.cfg, self.pattern, self.b = cfg, pattern, int(block_size)
        D.require_cuda()
        if cfg.jacobi_partitions > 0:
            self._phase = None       # (the relaxed operator depends on values)
            return
        n, bb = pattern.num_block_rows, self.b * self.b
        pat = D.DevPattern.upload(pattern)
        self.bsr = D.DevBSR(pat, self.b, torch.empty(max(pattern.num_blocks, 1) * bb,
                                                     dtype=torch.float64, device=pat.rp.device))
        stand = _PatternStandIn(pattern, self.b)
        plan = plan_device(cfg.backend, pat)
        prep = prepare_two_colour(stand, plan, pat)
        prep_g = prepare_general(stand, plan, pat) if prep is None else None
        if prep_g is not None:
            prep_g["persistent"] = True
        self._phase = (plan, prep, prep_g)
        self._n = n

    def close(self):
        phase, self._phase = getattr(self, "_phase", None), None
        if phase is None:
            return
        g = phase[2]
        if g is not None:
            if g.get("sym") is not None:
                D.lib().b2s_ilu0_symbolic_free(g["sym"], D.stream())
                g["sym"] = None
            if g.get("gw") is not None:
                D.lib().b2s_gw_destroy(g["gw"][0])
                g["gw"] = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _serves(self, a: BlockMatrix, wells) -> bool:
        if self._phase is None or a.block_size != self.b:
            return False
        if wells is not None and not wells.is_empty and self.cfg.well_mode is WellMode.COUPLED:
            return False
        p = a.pattern
        return p is self.pattern or (
            p.num_block_rows == self.pattern.num_block_rows
            and np.array_equal(p.row_pointers, self.pattern.row_pointers)
            and np.array_equal(p.column_indices, self.pattern.column_indices))

    def solve(self, a: BlockMatrix, b: BlockVector, wells=None,
              x0: BlockVector | None = None) -> tuple[BlockVector, SolveReport]:
        from .errors import ShapeError
        if not self._serves(a, wells):
            return solve_with_fallback(self.cfg, a, b, wells, x0)
        cfg = self.cfg
        a_sys = a.as_block_row_major()
        n, bs = a_sys.num_block_rows, a_sys.block_size
        if b.block_size != bs or b.num_blocks != n:
            raise ShapeError("right-hand side does not match the operator")
        if x0 is not None and (x0.block_size != bs or x0.num_blocks != n):
            raise ShapeError("initial guess does not match the right-hand side")
        sep = None
        if wells is not None and not wells.is_empty:
            sep = WellSet(wells.standard, wells.multisegment, WellMode.SEPARATE)
        t0 = time.perf_counter()
        dev = self.bsr.vals.device
        src = torch.from_numpy(a_sys.values)
        nv = src.numel()
        if D.is_pinned(src) or nv * 8 < D.STAGE_MIN_BYTES:
            self.bsr.vals[:nv].copy_(src, non_blocking=D.is_pinned(src))
        else:
            D.staged_copy(self.bsr.vals[:nv], src, torch.cuda.current_stream(dev))
        rhs = D.to_device(torch.from_numpy(np.ascontiguousarray(b.data, dtype=np.float64)), dev)
        x0d = (torch.zeros(n * bs, dtype=torch.float64, device=dev) if x0 is None
               else D.to_device(torch.from_numpy(np.ascontiguousarray(x0.data)), dev))
        try:
            solver = DeviceSolver(a_sys, self.bsr, cfg, wells=sep).setup(
                pattern_phase=self._phase)
            norm0 = RefNorm(_initial_residual(self.bsr, rhs, None if x0 is None else x0d, sep),
                            n * bs)
            e_setup = torch.cuda.Event(enable_timing=True)
            e_setup.record()
            xd = x0d.clone()
            queue = _Tail(xd, n * bs, bs, norm0)
            res = solver.solve(rhs, xd, cfg.stop, x0_zero=x0 is None, on_done=queue)
            e_end, tail = queue.wait()
            rep = _report(res, e_setup.elapsed_time(e_end) / 1e3, solver.plan.group_count,
                          norm0.from_tail(tail))
            rep.setup_elapsed = max((time.perf_counter() - t0) - rep.elapsed, 0.0)
        except SingularPivot:
            return solve_with_fallback(cfg, a, b, wells, x0)
        if not rep.converged:
            return solve_with_fallback(cfg, a, b, wells, x0)
        return tail.vector(), rep
