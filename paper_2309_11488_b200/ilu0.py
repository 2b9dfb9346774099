"""Zero-fill block ILU0 on the GPU: ``decompose`` and ``Ilu0Factorization``.

Same contract as ``bs/ilu0.py``: the factorisation runs on the plan-permuted
copy of the matrix in ascending permuted order (IKJ), keeps combined L\\U in
the input pattern (permuted), raises ``MissingDiagonal`` / ``SingularPivot``
with input row numbers, and ``apply`` solves L y = r, U z = y with the
permutation handled internally.

Device work (csrc/analysis.cu, csrc/ilu0.cu): permutation, sync-free
factorisation, then SELL-32 tiles of the strict-lower and strict-upper
blocks plus the inverse-diagonal tiles that the sweeps stream.  Host
attributes (``combined``, ``inverted_diagonals``) are materialised lazily.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

from . import _device as D
from ._lib import SINGULAR_PIVOT, UNSUPPORTED, check
from .analysis import ParallelPlan, apply_permutation, dev_to_matrix, permute_device
from .blockcore import BlockMatrix, BlockVector
from .errors import MissingDiagonal, ShapeError, SingularPivot


def _kc(width: int) -> int:
    """Register prefetch depth of the sweeps: wider rows are walked in chunks
    of 4 (8-deep chunks cost ~240 registers and halve the resident warps)."""
    return 2 if width <= 2 else 4


_I32_MAX = 2 ** 31 - 1


class Ilu0Factorization:
    """Combined L/U factors (plan order), inverse diagonals and the plan,
    resident on the GPU (bs/ilu0.py:59-142)."""

    def __init__(self, plan: ParallelPlan, b: int, n: int, lu: "D.DevBSR", invd: torch.Tensor,
                 smap: "D.SliceMap", lower: "D.Sell", upper: "D.Sell", dtiles: torch.Tensor,
                 identity: bool, source: BlockMatrix, a_perm: "D.DevBSR", two_colour=None):
        self.plan = plan
        self._b = b
        self._n = n
        self._lu = lu
        self._invd = invd
        self._deferred = None    # device flags of a not yet checked factorisation
        self._op_shell = None    # the operator's SELL layout, sized in the pattern phase
        self._gw_lazy = None     # wavefront factorisation: what materialises L\U on request
        self.smap = smap
        self._lower = lower
        self._upper = upper
        self.dtiles = dtiles
        self._identity_perm = identity
        self._source = source        # the (block-row-major) matrix that was factored
        self._a_perm = a_perm        # its unfactored plan-order copy (reused as operator)
        self._a_src = None           # or (plan-order pattern, source map, input BSR)
        # 2-colour plans (csrc/factor2c.cu): the operator's SELL layout (U's
        # rows live there) and what is needed to rebuild the CSR factors
        self._two_colour = two_colour
        self.a_sell = two_colour["a_sell"] if two_colour else None
        # (deep plans of grids take the wavefront sweeps, csrc/gridwave.cu: their
        # SELL layouts are built only if something asks for them)
        if lower is None:
            self.kc = 2
        else:
            uw = (self.a_sell.width - 1) if two_colour else upper.width
            self.kc = _kc(max(lower.width, uw))
        self._combined = None
        self._inv_host = None
        self._tickets = torch.zeros(8, dtype=torch.int32, device=invd.device)
        # measured on B200 (tools/sweep_bench.py): few groups (colourings) are
        # bandwidth-bound -> static slice order, no ticket atomics (0.77 of
        # peak vs 0.68); deep level schedules are latency-bound -> dynamic
        # tickets on one CTA of 4 warps per SM (fewer pollers on L2: C4 level
        # application 626 us vs 685 us with 8 warps, a warps-per-CTA scan, round 1)
        self.sweep_flags = 0x4 if plan.group_count <= 16 else 0x410
        self.tiles = None        # b2s_tiles_create handle (tiled level sweeps), or None
        self.gw = None           # b2s_gw_create handle (wavefront sweeps of grids), or None
        # few independent groups (colourings) and no same-group entries: the
        # phased sweeps, 2(G-1) plain passes, no polling (bit-identical)
        # (2(G-1) kernels per application: they pay for colourings -- few wide
        # groups -- while shallow level schedules of small systems are faster
        # on the sync-free sweeps: 13x7x9 level 286 vs 141 us per BiCGStab
        # iteration, 10x10x10 306 vs 141, profiles/r02/phased_small.txt)
        ng = len(smap.gslice_host) - 1 if smap.gslice_host is not None else 0
        self.phased = (smap.gslice_host is not None and lower is not None and not lower.stale
                       and not (False if two_colour else upper.stale)
                       and (ng <= 4 or self._n >= 4096 * ng)
                       and os.environ.get("B2S_PHASED", "1") != "0")

    def check_deferred(self) -> bool:
        """Read the flags of a deferred factorisation (synchronises): raises
        SingularPivot (input numbering, as decompose would have); True if a
        2-colour pattern was not a 2-colour structure after all (the caller
        refactorises with the general path).  False when nothing is pending."""
        fl, self._deferred = self._deferred, None
        if fl is None:
            return False
        bad, unsupported = (int(v) for v in fl.cpu().tolist())
        if unsupported:
            return True
        if bad != _I32_MAX:
            raise SingularPivot(int(self.plan.device("inverse_permutation")[bad].item()))
        return False

    # -- lazily materialised pieces of a 2-colour factorisation ----------------
    @property
    def lu_device(self) -> "D.DevBSR":
        """Combined L\\U in plan order, block CSR (built on first use for 2-colour
        factorisations, which never need it on the solve path)."""
        if self._lu is None and self._gw_lazy is not None:
            # wavefront factorisation: operator values in plan order, then the
            # L blocks and U_ii from the records written over them
            ppat, src, vin, diag, dvals = self._gw_lazy
            bb = self._b * self._b
            vals = D.empty_f64(max(ppat.nnz, 1) * bb, ppat.rp.device)
            if src is None:
                vals[: ppat.nnz * bb].copy_(vin[: ppat.nnz * bb])
            elif ppat.nnz:
                check(D.lib().b2s_gather_blocks(ppat.nnz, self._b, D.ptr(src), D.ptr(vin),
                                                D.ptr(vals), D.stream()), "gather_blocks")
            check(D.lib().b2s_gw_unpack_lu(self.gw, D.ptr(diag), D.ptr(dvals), D.ptr(vals),
                                           D.stream()), "gw_unpack_lu")
            self._lu = D.DevBSR(ppat, self._b, vals)
        if self._lu is None:
            t = self._two_colour
            pat, a_s, lo = t["pattern"], t["a_sell"], self.lower
            bb = self._b * self._b
            vals = D.empty_f64(pat.nnz * bb, pat.rp.device)
            check(D.lib().b2s_factor_2colour_combined(
                self._n, self._b, t["goff1"], t["s1"], D.ptr(pat.rp), D.ptr(a_s.sp),
                D.ptr(a_s.cols), D.ptr(a_s.vals), D.ptr(lo.sp), D.ptr(lo.cols), D.ptr(lo.vals),
                D.ptr(t["udiag"]), D.ptr(vals), D.stream()), "factor_2colour_combined")
            self._lu = D.DevBSR(pat, self._b, vals)
        return self._lu

    @property
    def lower(self) -> "D.Sell":
        if self._lower is None:
            self._lower = D.Sell.build(self.smap, self.lu_device, 1,
                                       self.plan.device("group_offsets"), self.plan.group_count)
        return self._lower

    @property
    def upper(self) -> "D.Sell":
        if self._upper is None:
            self._upper = D.Sell.build(self.smap, self.lu_device, 2,
                                       self.plan.device("group_offsets"), self.plan.group_count)
        return self._upper

    # -- reference attributes --------------------------------------------------
    @property
    def block_size(self) -> int:
        return self._b

    @property
    def num_block_rows(self) -> int:
        return self._n

    @property
    def combined(self) -> BlockMatrix:
        if self._combined is None:
            if self._identity_perm:
                bb = self._b * self._b
                vals = self.lu_device.vals[: self.lu_device.pat.nnz * bb].cpu().numpy()
                self._combined = BlockMatrix(self._source.pattern, self._b, vals)
            else:
                self._combined = dev_to_matrix(self.lu_device)
        return self._combined

    @property
    def inverted_diagonals(self) -> np.ndarray:
        if self._inv_host is None:
            bb = self._b * self._b
            self._inv_host = self._invd[: self._n * bb].cpu().numpy().reshape(self._n, self._b,
                                                                             self._b)
        return self._inv_host

    def factors_in_input_order(self) -> BlockMatrix:
        """The combined factors carried back to input numbering (bs/ilu0.py:79-83)."""
        if self._identity_perm:
            return self.combined.copy()
        return dev_to_matrix(permute_device(self.lu_device, self.plan, inverse=True))

    # -- application -------------------------------------------------------------
    def apply_device(self, r_perm: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """z = U^-1 L^-1 r for a plan-order device vector."""
        m = self._n * self._b
        dev = r_perm.device
        y = D.empty_f64(m, dev)
        z = out if out is not None else D.empty_f64(m, dev)
        if m == 0:
            return z
        s, lo, up = self.smap, self.lower, self.upper
        if self.phased and not self.tiles:
            check(D.lib().b2s_ilu0_apply_phased(
                self._n, self._b, self.kc, len(s.gslice_host) - 1,
                s.gslice_host.ctypes.data, s.goff1, D.ptr(s.row0), D.ptr(s.nrows),
                D.ptr(lo.sp), D.ptr(lo.cols), D.ptr(lo.vals), D.ptr(up.sp), D.ptr(up.cols),
                D.ptr(up.vals), D.ptr(self.dtiles), D.ptr(r_perm), D.ptr(y), D.ptr(z),
                D.stream()), "ilu0_apply_phased")
            return z
        if self.gw:
            check(D.lib().b2s_gw_apply(self._b, self.gw, D.ptr(r_perm), D.ptr(z), D.stream()),
                  "gw_apply")
            return z
        D.fill_sentinel(y, m)
        D.fill_sentinel(z, m)
        if self.tiles:
            check(D.lib().b2s_tiles_apply(self._b, self.tiles, D.ptr(r_perm), D.ptr(y), D.ptr(z),
                                          0 if self.upper.stale else 1, D.stream()),
                  "tiles_apply")
            return z
        s = self.smap
        lo, up = self.lower, self.upper
        check(D.lib().b2s_ilu0_apply(self._n, self._b, self.kc, s.nslices, D.ptr(s.row0),
                                     D.ptr(s.nrows), D.ptr(lo.sp), D.ptr(lo.cols),
                                     D.ptr(lo.vals), D.ptr(up.sp), D.ptr(up.cols),
                                     D.ptr(up.vals), D.ptr(self.dtiles), D.ptr(r_perm),
                                     D.ptr(y), D.ptr(z), 0 if self.upper.stale else 1,
                                     self.sweep_flags, D.ptr(self._tickets), D.stream()),
              "ilu0_apply")
        return z

    def apply(self, r: BlockVector) -> BlockVector:
        if r.block_size != self._b:
            raise ShapeError("vector block size does not match factorization")
        if r.num_blocks != self._n:
            raise ShapeError("vector length does not match factorization")
        return BlockVector(self.apply_array(r.data), self._b)

    def apply_array(self, r: np.ndarray) -> np.ndarray:
        """Input order in, input order out (bs/ilu0.py:93-103)."""
        if self._n == 0:
            return np.asarray(r, dtype=np.float64).copy()
        dev = self._invd.device
        rd = D.f64(np.asarray(r).reshape(-1), dev)
        if self._identity_perm:
            return self.apply_device(rd)[: self._n * self._b].cpu().numpy()
        rp = D.gather_rows(rd, self.plan.device("inverse_permutation"), self._n, self._b)
        z = self.apply_device(rp)
        return D.gather_rows(z, self.plan.device("permutation"), self._n,
                             self._b).cpu().numpy()

    def apply_permuted_array(self, r: np.ndarray) -> np.ndarray:
        if self._n == 0:
            return np.asarray(r, dtype=np.float64).copy()
        rd = D.f64(np.asarray(r).reshape(-1), self._invd.device)
        return self.apply_device(rd)[: self._n * self._b].cpu().numpy()

    def __call__(self, r: np.ndarray) -> np.ndarray:
        return self.apply_array(r)

    def __del__(self):
        if getattr(self, "gw", None) and getattr(self, "_gw_owner", True):
            try:
                D.lib().b2s_gw_destroy(self.gw)
            except Exception:
                pass
            self.gw = None
        if getattr(self, "tiles", None):
            try:
                D.lib().b2s_tiles_destroy(self.tiles)
            except Exception:
                pass
            self.tiles = None


def prepare_two_colour(a: BlockMatrix, plan: ParallelPlan, pat: "D.DevPattern"):
    """Pattern-only half of the 2-colour factorisation (permuted pattern and
    source map, slice map, layout offsets, buffers): runs while the values
    are still on their way to the device.  None when the plan is not a
    2-group plan this path handles."""
    n, b = a.num_block_rows, a.block_size
    if not (plan.group_count == 2 and not plan.is_identity and b <= 4 and
            os.environ.get("B2S_FACTOR_2C", "1") != "0"):
        return None
    D.find_diagonal(pat)                           # MissingDiagonal(first row)
    bb = b * b
    dev = pat.rp.device
    ppat, src = D.permute_pattern(pat, plan.device("permutation"),
                                  plan.device("inverse_permutation"))
    smap = plan.slice_map()
    if smap.gslice_host is None or len(smap.gslice_host) != 3:
        return None
    shell = D.DevBSR(ppat, b, D.empty_f64(1, dev))     # pattern only
    return {"pattern": ppat, "src": src, "smap": smap,
            "a_sell": D.Sell.build(smap, shell, 0, fill=False),
            "lower": D.Sell.build(smap, shell, 1, fill=False),
            "inv": D.empty_f64(n * bb, dev),
            "udiag": D.empty_f64((n - int(smap.goff1)) * bb, dev),
            "dtiles": D.empty_f64(smap.nslices * bb * 32, dev),
            "s1": int(smap.gslice_host[1]), "goff1": int(smap.goff1)}


def _factor_two_colour(a: BlockMatrix, plan: ParallelPlan, bsr: "D.DevBSR", prep=None,
                       defer: bool = False):
    """2-colour plans: operator layout + factors straight from the input
    values (csrc/factor2c.cu); None if the pattern is not a 2-colour
    structure (then the general path runs).  ``defer``: no host read here --
    the singular-pivot / structure flags stay on the device until
    ``check_deferred()`` (the solve path reads them after its loop, so the
    host prepares the Krylov loop while the device factorises)."""
    n, b = a.num_block_rows, a.block_size
    prep = prep or prepare_two_colour(a, plan, bsr.pat)
    if prep is None:
        return None
    smap, a_sell, lower = prep["smap"], prep["a_sell"], prep["lower"]
    inv, udiag, dtiles = prep["inv"], prep["udiag"], prep["dtiles"]
    s1, goff1 = prep["s1"], prep["goff1"]
    a_sell.fill_from(smap, D.DevBSR(prep["pattern"], b, bsr.vals), 0, prep["src"])
    tc = {"pattern": prep["pattern"], "a_sell": a_sell, "udiag": udiag, "goff1": goff1, "s1": s1}
    if defer:
        flags = torch.full((2,), _I32_MAX, dtype=torch.int32, device=inv.device)
        flags[1:].zero_()
        check(D.lib().b2s_factor_2colour_async(
            n, b, goff1, s1, smap.nslices, D.ptr(smap.row0), D.ptr(smap.nrows),
            D.ptr(a_sell.sp), D.ptr(a_sell.cols), D.ptr(a_sell.vals), D.ptr(lower.sp),
            D.ptr(lower.cols), D.ptr(lower.vals), D.ptr(inv), D.ptr(udiag), D.ptr(dtiles),
            D.ptr(flags), D.stream()), "factor_2colour_async")
        f = Ilu0Factorization(plan, b, n, None, inv, smap, lower, None, dtiles, False, a, None,
                              two_colour=tc)
        f._deferred = flags
        return f
    bad = C.c_int32(-1)
    rc = D.lib().b2s_factor_2colour(n, b, goff1, s1, smap.nslices, D.ptr(smap.row0),
                                    D.ptr(smap.nrows), D.ptr(a_sell.sp), D.ptr(a_sell.cols),
                                    D.ptr(a_sell.vals), D.ptr(lower.sp), D.ptr(lower.cols),
                                    D.ptr(lower.vals), D.ptr(inv), D.ptr(udiag), D.ptr(dtiles),
                                    C.byref(bad), D.stream())
    if rc == UNSUPPORTED:
        return None
    if rc == SINGULAR_PIVOT:
        raise SingularPivot(int(plan.device("inverse_permutation")[int(bad.value)].item()))
    check(rc, "factor_2colour")
    return Ilu0Factorization(plan, b, n, None, inv, smap, lower, None, dtiles, False, a, None,
                             two_colour=tc)


def _gw_factor_on() -> bool:
    return os.environ.get("B2S_GW_FACTOR", "1") != "0"


def _symbolic(n: int, b: int, ppat: "D.DevPattern", diag: torch.Tensor):
    sym = C.c_void_p(None)
    check(D.lib().b2s_ilu0_symbolic(n, b, D.ptr(ppat.rp), D.ptr(ppat.ci), D.ptr(diag),
                                    C.byref(sym), D.stream()), "ilu0_symbolic")
    return sym


def _factor_gw(a: BlockMatrix, plan: ParallelPlan, bsr: "D.DevBSR", g: dict, defer: bool):
    """Wavefront factorisation of a natural-order grid (csrc/gridwave.cu
    b2s_gw_factor): straight from the input values into the sweep records;
    None when it declines (then the general numeric factorisation runs)."""
    n, b = a.num_block_rows, a.block_size
    bb = b * b
    identity, ppat, src, gw, diag, smap = (g["identity"], g["pattern"], g["src"], g["gw"],
                                           g["diag"], g["smap"])
    h = gw[0]
    dev = bsr.pat.rp.device
    nbytes = int(D.lib().b2s_gw_factor_workspace_bytes(h))
    ws = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=dev)
    inv = D.empty_f64(n * bb, dev)
    dvals = D.empty_f64(n * bb, dev)
    flags = torch.full((2,), _I32_MAX, dtype=torch.int32, device=dev)
    flags[1:].zero_()
    rc = D.lib().b2s_gw_factor(h, D.ptr(ppat.rp), D.ptr(ppat.ci), D.ptr(diag),
                               None if src is None else D.ptr(src), D.ptr(bsr.vals), D.ptr(inv),
                               D.ptr(dvals), D.ptr(flags), D.ptr(ws), nbytes, D.stream())
    if rc == UNSUPPORTED:
        return None
    check(rc, "gw_factor")
    if not defer:
        bad = int(flags[0].item())
        if bad != _I32_MAX:
            raise SingularPivot(bad if identity else
                                int(plan.device("inverse_permutation")[bad].item()))
    dtiles = D.empty_f64(smap.nslices * bb * 32, dev)
    check(D.lib().b2s_diag_tiles(smap.nslices, b, D.ptr(smap.row0), D.ptr(smap.nrows),
                                 D.ptr(inv), D.ptr(dtiles), D.stream()), "diag_tiles")
    f = Ilu0Factorization(plan, b, n, None, inv, smap, None, None, dtiles, identity, a,
                          bsr if identity else None)
    f._a_src = None if identity else (ppat, src, bsr)
    f._op_shell = g["op_shell"]
    f._deferred = flags if defer else None
    f._gw_lazy = (ppat, src, bsr.vals, diag, dvals)
    f.gw, f._gw_ws, f.gw_shape = gw
    f._gw_owner = not g.get("persistent")
    return f


def prepare_general(a: BlockMatrix, plan: ParallelPlan, pat: "D.DevPattern"):
    """Pattern-only half of the general factorisation: plan-order pattern and
    source map, diagonal positions, slice map, the symbolic factorisation
    (update pairs), the wavefront packing's pattern phase and the operator's
    SELL layout (sized, filled later).  Every host synchronisation of the
    setup that depends on the pattern alone happens here -- before the values
    are needed (the solve path runs it while they are still uploading)."""
    n, b = a.num_block_rows, a.block_size
    D.find_diagonal(pat)                           # MissingDiagonal(first row)
    identity = plan.is_identity
    if identity:
        ppat, src = pat, None
    else:
        # plan-order pattern + source map; the factor's values are gathered
        # straight from the input (one pass), and the operator layout is
        # later filled from the input the same way -- no permuted copy
        ppat, src = D.permute_pattern(pat, plan.device("permutation"),
                                      plan.device("inverse_permutation"))
    gw = _gw_plan(pat.grid, plan, ppat, b)
    diag = D.find_diagonal(ppat)
    # group-aligned slices: a sweep never waits on a row of its own group
    # (same-group reads take the pre-sweep value, as the reference does)
    smap = plan.slice_map()
    # (the wavefront factorisation needs no update pairs; they are computed
    # later only if it declines)
    sym = None if (gw is not None and _gw_factor_on()) else _symbolic(n, b, ppat, diag)
    shell = D.DevBSR(ppat, b, D.empty_f64(1, ppat.rp.device))   # pattern only
    return {"identity": identity, "pattern": ppat, "src": src, "gw": gw, "diag": diag,
            "smap": smap, "sym": sym, "op_shell": D.Sell.build(smap, shell, 0, fill=False)}


def factor_device(a: BlockMatrix, plan: ParallelPlan, bsr: "D.DevBSR" = None,
                  prep=None, defer: bool = False, two_colour: bool = True,
                  prep_general=None) -> Ilu0Factorization:
    """``decompose`` on an (optionally pre-uploaded) matrix; ``prep`` /
    ``prep_general``: ``prepare_two_colour`` / ``prepare_general``'s
    pattern-only half when the caller ran it early.  ``defer``: no host read
    of the pivot check (the caller must call ``check_deferred()`` before
    trusting any result); ``two_colour=False`` forces the general
    factorisation."""
    a = a.as_block_row_major()
    n = a.num_block_rows
    if plan.num_rows != n:
        raise ShapeError("plan does not match the matrix")
    b = a.block_size
    bsr = bsr or D.DevBSR.upload(a)
    dev = bsr.pat.rp.device
    f = (_factor_two_colour(a, plan, bsr, prep, defer)
         if two_colour and prep_general is None else None)
    if f is not None:
        return f
    g = prep_general or prepare_general(a, plan, bsr.pat)
    if g["gw"] is not None and _gw_factor_on():
        f = _factor_gw(a, plan, bsr, g, defer)
        if f is not None:
            return f
    if g["sym"] is None:
        g["sym"] = _symbolic(n, b, g["pattern"], g["diag"])
    identity, ppat, src, gw = g["identity"], g["pattern"], g["src"], g["gw"]
    diag, smap, sym = g["diag"], g["smap"], g["sym"]
    a_src = None
    if identity:
        a_perm = bsr
        lu = D.DevBSR(bsr.pat, b, bsr.vals.clone())
    else:
        vals = D.empty_f64(bsr.pat.nnz * b * b, dev)
        if bsr.pat.nnz:
            check(D.lib().b2s_gather_blocks(bsr.pat.nnz, b, D.ptr(src), D.ptr(bsr.vals),
                                            D.ptr(vals), D.stream()), "gather_blocks")
        lu = D.DevBSR(ppat, b, vals)
        a_perm, a_src = None, (ppat, src, bsr)
    inv = D.empty_f64(n * b * b, dev)
    flags = None
    try:
        if defer:
            flags = torch.full((2,), _I32_MAX, dtype=torch.int32, device=dev)
            flags[1:].zero_()
            rc = D.lib().b2s_ilu0_numeric(sym, b, smap.nslices, D.ptr(smap.row0),
                                          D.ptr(smap.nrows), D.ptr(lu.pat.rp), D.ptr(lu.pat.ci),
                                          D.ptr(diag), D.ptr(lu.vals), D.ptr(inv), D.ptr(flags),
                                          None, D.stream())
        else:
            bad = C.c_int32(-1)
            rc = D.lib().b2s_ilu0_numeric(sym, b, smap.nslices, D.ptr(smap.row0),
                                          D.ptr(smap.nrows), D.ptr(lu.pat.rp), D.ptr(lu.pat.ci),
                                          D.ptr(diag), D.ptr(lu.vals), D.ptr(inv), None,
                                          C.byref(bad), D.stream())
            if rc == SINGULAR_PIVOT:
                row = int(bad.value)
                if not identity:
                    row = int(plan.device("inverse_permutation")[row].item())
                raise SingularPivot(row)
        check(rc, "ilu0_numeric")
    finally:
        if not g.get("persistent"):   # (a SolveSession keeps it for the next values)
            D.lib().b2s_ilu0_symbolic_free(sym, D.stream())
            g["sym"] = None
    goff = plan.device("group_offsets")
    lower = upper = None
    if gw is None:   # (the wavefront sweeps read their own packed records)
        lower = D.Sell.build(smap, lu, 1, goff, plan.group_count)
        upper = D.Sell.build(smap, lu, 2, goff, plan.group_count)
    dtiles = D.empty_f64(smap.nslices * b * b * 32, dev)
    check(D.lib().b2s_diag_tiles(smap.nslices, b, D.ptr(smap.row0), D.ptr(smap.nrows),
                                 D.ptr(inv), D.ptr(dtiles), D.stream()), "diag_tiles")
    f = Ilu0Factorization(plan, b, n, lu, inv, smap, lower, upper, dtiles, identity, a, a_perm)
    f._a_src = a_src
    f._op_shell = g["op_shell"]
    f._deferred = flags
    _maybe_tiles(f, plan, diag)
    _gw_fill(f, gw)
    f._gw_owner = not g.get("persistent")
    return f


def grid_shape(a: BlockMatrix):
    """(nx, ny, nz) if ``a`` looks like a natural-order 3D 7-point grid (all
    off-diagonal couplings at offsets 1, nx, nx*ny), else None.  Only used to
    shape the sweep tiles; results never depend on it."""
    p = a.pattern
    n = p.num_block_rows
    m = min(n, 65536)
    if m < 8:
        return None
    end = int(p.row_pointers[m])
    rows = np.repeat(np.arange(m, dtype=np.int64), np.diff(p.row_pointers[: m + 1]))
    off = np.abs(p.column_indices[:end] - rows)
    u = np.unique(off[off > 0])
    if len(u) != 3 or u[0] != 1 or u[2] % u[1] or n % u[2]:
        return None
    nx, nxy = int(u[1]), int(u[2])
    return nx, nxy // nx, n // nxy


def _patches(nx: int, ny: int, tiles: int):
    """px x py <= tiles column patches, as square as the grid allows."""
    cands = []
    for px in range(1, min(nx, tiles) + 1):
        py = min(ny, tiles // px)
        if py >= 1:
            cands.append((px * py, abs(nx / px - ny / py), px, py))
    most = max(c[0] for c in cands)
    # near-maximal tile count, then the squarest patches (fewest boundary rows)
    ok = [c for c in cands if c[0] >= 0.9 * most]
    _, _, px, py = min(ok, key=lambda c: (c[1], -c[0]))
    return px, py


def _gw_tile_shape(nx: int, ny: int) -> tuple[int, int]:
    """Columns of one wavefront tile (one warp: wx * wy <= 32): 8 x 4 keeps
    the tile crossings on the critical path (TX + TY) low at 1M cells."""
    env = os.environ.get("B2S_GW_TILE")
    if env:
        wx, wy = (int(v) for v in env.split(","))
        return min(wx, nx), min(wy, ny)
    wx = min(nx, 8)
    wy = max(1, min(ny, 32 // wx))
    return wx, wy


def _gw_plan(hint, plan: ParallelPlan, ppat: "D.DevPattern", b: int):
    """Pattern phase of the wavefront sweeps (csrc/gridwave.cu) for deep plans
    of a natural-order 7-point grid: one warp per tile of columns, in-tile
    dependencies through warp shuffles, bit-identical to the sync-free
    sweeps.  Runs before the numeric factorisation is queued (its single
    synchronisation waits for the pattern work only); the kernel checks every
    row, anything else keeps the sync-free sweeps.  Returns (handle,
    workspace, shape) or None.  ``hint``: the input pattern's grid_hint
    (nx, ny) -- taken at upload from one row; the kernel verifies them all.
    B2S_GW=0 turns it off."""
    if os.environ.get("B2S_GW", "1") == "0" or os.environ.get("B2S_TILES", "0") != "0":
        return None
    if plan.group_count <= D.PHASED_MAX_GROUPS or b > 4:
        return None
    n = ppat.n
    if hint is None or n % (hint[0] * hint[1]):
        return None
    nx, ny = hint
    nz = n // (nx * ny)
    wx, wy = _gw_tile_shape(nx, ny)
    nbytes = int(D.lib().b2s_gw_workspace_bytes(n, b, nx, ny, nz, wx, wy))
    if nbytes <= 0:
        return None
    # the packed factor lives in a caching-allocator block (no cudaMalloc per solve)
    ws = torch.empty(nbytes // 8 + 1, dtype=torch.float64, device=ppat.rp.device)
    h = C.c_void_p(None)
    rc = D.lib().b2s_gw_create(n, b, nx, ny, nz, wx, wy, D.ptr(plan.device("permutation")),
                               D.ptr(plan.device("inverse_permutation")), D.ptr(ppat.rp),
                               D.ptr(ppat.ci), D.ptr(ws), nbytes, C.byref(h), D.stream())
    if rc == 5:   # B2S_UNSUPPORTED: not a stencil row of this plan / too many tiles
        return None
    check(rc, "gw_create")
    return h.value, ws, (nx, ny, nz, wx, wy)


def _gw_fill(f: Ilu0Factorization, gw):
    """Value phase: the factor's blocks into the step records (async)."""
    if gw is None:
        return
    h, ws, shape = gw
    f.gw, f._gw_ws, f.gw_shape = h, ws, shape
    check(D.lib().b2s_gw_fill(h, D.ptr(f._lu.vals), D.ptr(f._invd), D.stream()), "gw_fill")


def _maybe_tiles(f: Ilu0Factorization, plan: ParallelPlan, diag: torch.Tensor):
    """Opt-in (B2S_TILES=1): the tiled step kernels (csrc/tiles.cu), which
    resolve in-tile dependencies of a level schedule on-chip.  Results are
    bit-identical to the sync-free sweeps, but on B200 they are not faster yet
    (C4: 0.87 ms vs 0.68 ms per application; profiles/r01/tile_steps_trace.json,
    DESIGN.md section 3), so the sync-free sweeps stay the default.
    B2S_TILES_T sets the tile count (default: the SMs, or the column patches
    of a natural-order grid that fit on them)."""
    if os.environ.get("B2S_TILES", "0") == "0":
        return
    n = f.num_block_rows
    sms = torch.cuda.get_device_properties(diag.device).multi_processor_count
    T = int(os.environ.get("B2S_TILES_T", sms))
    min_rows = int(os.environ.get("B2S_TILES_MIN_ROWS", 64))     # per tile
    if plan.group_count < int(os.environ.get("B2S_TILES_MIN_GROUPS", 32)) or n < min_rows * T:
        return
    nx = ny = px = py = 0
    g = grid_shape(f._source) if os.environ.get("B2S_TILES_GRID", "1") == "1" else None
    if g is not None and g[2] > 1:
        nx, ny, _ = g
        px, py = _patches(nx, ny, T)
    h = C.c_void_p(None)
    rc = D.lib().b2s_tiles_create(n, f._b, T, nx, ny, px, py,
                                  D.ptr(plan.device("inverse_permutation")),
                                  D.ptr(f.lu_device.pat.rp), D.ptr(f.lu_device.pat.ci), D.ptr(diag),
                                  D.ptr(f.lu_device.vals), D.ptr(f._invd),
                                  D.ptr(plan.device("group_offsets")), plan.group_count,
                                  C.byref(h), D.stream())
    if rc == 5:   # B2S_UNSUPPORTED: the ring does not fit, keep the sync-free sweeps
        return
    check(rc, "tiles_create")
    f.tiles = h.value
    f.tile_shape = (px, py) if px else (T,)


def decompose(a: BlockMatrix, plan: ParallelPlan) -> Ilu0Factorization:
    """Blocked zero-fill LU of ``a`` in plan order (bs/ilu0.py:145-201)."""
    a = a.as_block_row_major()
    if plan.num_rows != a.num_block_rows:
        raise ShapeError("plan does not match the matrix")
    return factor_device(a, plan)


__all__ = ["Ilu0Factorization", "decompose", "apply_permutation"]
