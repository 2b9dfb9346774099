"""Multi-GPU ILU0-BiCGStab: contiguous row slabs, block-Jacobi ILU0, halo
SpMV and all-reduced inner products (the paper's MPI
decomposition).

Each rank ("shard") owns a contiguous range of global rows -- a z-slab of
the natural-order grid.  Its preconditioner is ILU0 of the diagonal block
(cross-slab couplings dropped, exactly ``drop_cross_blocks`` with the slab
partition, bs/jacobi.py:111-136), so factorisation and sweeps are local.
The operator keeps every coupling: before each SpMV the ghost rows (the
off-slab columns a shard references) are exchanged with the owning ranks.
The BiCGStab control flow is the reference's (bs/krylov.py:171-244); its
scalars are sums of per-shard partials combined by an all-reduce, so every
rank takes identical decisions.

Communication is behind a small interface with two implementations:
``NcclComm`` (one shard per process, torch.distributed over NCCL/NVLink,
halos by grouped send/recv) and ``LocalComm`` (several shards in one
process on one GPU, device copies and host sums) -- the latter lets the
partitioned solver be checked against the oracle on a single GPU.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from ._lib import check
from .analysis import ParallelPlan
from .blockcore import BlockMatrix, Layout, SparsityPattern
from .bridge import Backend, plan_device
from .ilu0 import factor_device
from .krylov import _BREAKDOWN_FLOOR, SolveReport, StoppingCriteria
from .synthetic import GeneratorSpec


# ---------------------------------------------------------------------------
# slab generation: the rows [r0, r1) of generate(spec), without the rest

@dataclass
class Slab:
    rank: int
    world: int
    n_global: int
    r0: int
    r1: int
    b: int
    rp: np.ndarray        # local rows, int64
    ci: np.ndarray        # GLOBAL column ids, int64
    vals3: np.ndarray     # (nnz, b, b)
    rhs: np.ndarray       # (r1 - r0) * b

    @property
    def rows(self) -> int:
        return self.r1 - self.r0


def slab_bounds(nz: int, world: int, rank: int) -> tuple[int, int]:
    """z-planes [z0, z1) of a rank: equal shares, the first ranks take the rest."""
    base, rem = divmod(nz, world)
    z0 = rank * base + min(rank, rem)
    return z0, z0 + base + (1 if rank < rem else 0)


def generate_slab(spec: GeneratorSpec, rank: int, world: int) -> Slab:
    """Rows of the z-planes [z0, z1) of ``generate(spec)``, bit-identical to
    the corresponding rows of the full system: the same PCG64 stream is
    advanced past the draws other slabs own (bs/io.py:363-414 draw order:
    all +x, +y, +z couplings src->dst in meshgrid order, then their mirrors,
    then the right-hand side)."""
    nx, ny, nz, b = spec.nx, spec.ny, spec.nz, spec.block_size
    bb = b * b
    nxy = nx * ny
    n = nxy * nz
    z0, z1 = slab_bounds(nz, world, rank)
    nfx, nfy, nfz = (nx - 1) * ny * nz, nx * (ny - 1) * nz, nxy * (nz - 1)
    npairs = nfx + nfy + nfz
    # runs of consecutive coupling indices this slab needs: (first, count,
    # direction, forward?) -- iz is the fastest enumeration index
    runs = []
    for fwd in (True, False):
        base = 0 if fwd else npairs
        for ix in range(nx - 1):                       # +x faces
            for iy in range(ny):
                e0 = (ix * ny + iy) * nz
                runs.append((base + e0 + z0, z1 - z0, "x", fwd, ix, iy, z0))
        for ix in range(nx):                           # +y faces
            for iy in range(ny - 1):
                e0 = nfx + (ix * (ny - 1) + iy) * nz
                runs.append((base + e0 + z0, z1 - z0, "y", fwd, ix, iy, z0))
        for ix in range(nx):                           # +z faces
            for iy in range(ny):
                e0 = nfx + nfy + (ix * ny + iy) * (nz - 1)
                # forward block rows = src (iz); backward rows = dst (iz + 1)
                lo, hi = (z0, min(z1, nz - 1)) if fwd else (max(z0 - 1, 0), z1 - 1)
                if hi > lo:
                    runs.append((base + e0 + lo, hi - lo, "z", fwd, ix, iy, lo))
    runs.sort(key=lambda r: r[0])
    rng = np.random.default_rng(spec.seed)
    bg = rng.bit_generator
    pos = 0
    rows_l, cols_l, blks_l = [], [], []
    tdir = {"x": spec.tx, "y": spec.ty, "z": spec.tz}
    step = {"x": 1, "y": nx, "z": nxy}
    for first, count, d, fwd, ix, iy, iz0 in runs:
        if first * bb > pos:
            bg.advance(first * bb - pos)
            pos = first * bb
        u = rng.uniform(0.5, 1.5, size=(count, b, b))
        pos += count * bb
        iz = iz0 + np.arange(count, dtype=np.int64)
        src = ix + nx * (iy + ny * iz)
        dst = src + step[d]
        rows_l.append(src if fwd else dst)
        cols_l.append(dst if fwd else src)
        blks_l.append(-tdir[d] * u)
    rhs_first = 2 * npairs * bb + z0 * nxy * b
    bg.advance(rhs_first - pos)
    rhs = rng.uniform(-1.0, 1.0, size=(z1 - z0) * nxy * b)
    r0, r1 = z0 * nxy, z1 * nxy
    diag = np.arange(r0, r1, dtype=np.int64)
    rows = np.concatenate(rows_l + [diag])
    cols = np.concatenate(cols_l + [diag])
    blk = np.concatenate(blks_l + [np.zeros((r1 - r0, b, b))])
    order = np.lexsort((cols, rows))
    rows, cols, blk = rows[order], cols[order], blk[order]
    nloc = r1 - r0
    rp = np.zeros(nloc + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows - r0, minlength=nloc), out=rp[1:])
    sums = np.zeros((nloc, b))
    np.add.at(sums, rows - r0, np.abs(blk).sum(axis=2))
    dpos = np.flatnonzero(rows == cols)
    eye = np.arange(b)
    dblk = np.zeros((nloc, b, b))
    dblk[:, eye, eye] = sums + spec.diagonal_boost
    blk[dpos] = dblk
    return Slab(rank, world, n, r0, r1, b, rp, cols, blk, rhs)


# ---------------------------------------------------------------------------
# one rank's device state

class HaloPlan:
    """Host-side halo bookkeeping of one slab (pure numpy): the ghost rows it
    references, which rank owns each, and local column ids with the ghosts
    appended after the owned rows."""

    def __init__(self, slab: Slab, owners: np.ndarray):
        self.slab = slab
        R = slab.rows
        ci = slab.ci
        self.own = (ci >= slab.r0) & (ci < slab.r1)
        self.ghosts = np.unique(ci[~self.own])          # global ids, ascending
        self.G = len(self.ghosts)
        gowner = np.searchsorted(owners, self.ghosts, side="right") - 1
        self.recv = {int(h): np.flatnonzero(gowner == h) for h in np.unique(gowner)}
        self.lcol = np.where(self.own, ci - slab.r0,
                             R + np.searchsorted(self.ghosts, ci)).astype(np.int64)

    def requests(self):
        """{owner rank: global ids this slab needs from it}"""
        return {h: self.ghosts[idx] for h, idx in self.recv.items()}


class _DeviceBlock:
    """A shard's diagonal block as the factorisation sees it: block size and
    pattern, with the values resident on the device only (gathered there from
    the uploaded slab) and the host pattern downloaded only if something asks
    for it -- no host copy of the slab's blocks, no host pattern pass."""

    def __init__(self, pat: "D.DevPattern", block_size: int):
        self._pat = pat
        self._pattern = None
        self.block_size = block_size
        self.layout = Layout.BLOCK_ROW_MAJOR

    @property
    def num_block_rows(self) -> int:
        return self._pat.n

    @property
    def pattern(self) -> SparsityPattern:
        if self._pattern is None:
            rp, ci = self._pat.host()
            self._pattern = SparsityPattern(self._pat.n, rp, ci)
        return self._pattern

    def as_block_row_major(self):
        return self

    @property
    def values(self):
        raise RuntimeError("a shard's preconditioner blocks live on the device only")


class _DeviceHalo:
    """The shard's halo bookkeeping computed on the device from the uploaded
    slab pattern (the host keeps only the ghost ids and their owners -- tens
    of thousands of ints): HaloPlan's result without its host passes over
    every coupling."""

    def __init__(self, ghosts: np.ndarray, recv: dict):
        self.ghosts, self.recv = ghosts, recv
        self.G = len(ghosts)

    def requests(self):
        """{owner rank: global ids this slab needs from it}"""
        return {h: self.ghosts[idx] for h, idx in self.recv.items()}


def _slab_grid_hint(slab: Slab):
    """grid_hint of the slab's diagonal block from its middle row (host, one row)."""
    R = slab.rows
    if R < 8:
        return None
    r = R // 2
    cols = np.asarray(slab.ci[int(slab.rp[r]):int(slab.rp[r + 1])], dtype=np.int64) - slab.r0
    cols = cols[(cols >= 0) & (cols < R)]
    u = [int(v) for v in np.unique(cols[cols > r] - r)]
    if u == [1]:
        return R, 1
    if len(u) == 2 and u[0] == 1 and R % u[1] == 0:
        return u[1], R // u[1]
    if len(u) == 3 and u[0] == 1 and u[2] % u[1] == 0 and R % u[2] == 0:
        return u[1], u[2] // u[1]
    return None


class Shard:
    """Local rows in plan order + ghost section, block-Jacobi ILU0, halo maps."""

    def __init__(self, slab: Slab, owners: np.ndarray, backend: Backend):
        self.slab = slab
        dev = D.require_cuda()
        R, b = slab.rows, slab.b
        self.R, self.b = R, b
        nnz = len(slab.ci)
        # one upload of the slab (pattern + values); the halo bookkeeping, the
        # diagonal block's pattern and its values are derived on the device
        # and stay resident -- setup() re-runs the device pipeline (plan,
        # permutation, factorisation, layouts) from them
        src = torch.from_numpy(np.ascontiguousarray(slab.ci, dtype=np.int64))
        ci = src.to(dev, non_blocking=D.is_pinned(src))
        rp32 = D.i32(slab.rp, dev)
        own = (ci >= slab.r0) & (ci < slab.r1)
        gh = ~own
        ghosts_d = torch.unique(ci[gh])                      # global ids, ascending
        lcol = torch.where(own, ci - slab.r0, R + torch.searchsorted(ghosts_d, ci))
        counts = (rp32[1:R + 1] - rp32[:R]).long()
        rows = torch.repeat_interleave(torch.arange(R, device=dev), counts, output_size=nnz)
        ghosts = ghosts_d.cpu().numpy()
        gowner = np.searchsorted(owners, ghosts, side="right") - 1
        recv = {int(h): np.flatnonzero(gowner == h) for h in np.unique(gowner)}
        self.halo_plan = _DeviceHalo(ghosts, recv)
        self.ghosts, self.G, self.recv = ghosts, len(ghosts), recv
        opat = D.DevPattern(R, nnz, rp32, lcol.to(torch.int32) if nnz else D.empty_i32(1, dev))
        self.obsr = D.DevBSR(opat, b, D.f64(slab.vals3.reshape(-1), dev))
        # preconditioner source: the diagonal block (cross-slab blocks dropped)
        own_rows = rows[own]
        prp = torch.zeros(R + 1, dtype=torch.int64, device=dev)
        prp[1:] = torch.cumsum(torch.bincount(own_rows, minlength=R), 0)
        self._own_idx = torch.nonzero(own).flatten().to(torch.int32)
        pnnz = int(self._own_idx.numel())
        ppat = D.DevPattern(R, pnnz, prp.to(torch.int32),
                            lcol[own].to(torch.int32) if pnnz else D.empty_i32(1, dev),
                            _slab_grid_hint(slab))
        self.pmat = _DeviceBlock(ppat, b)
        self.pbsr = D.DevBSR(ppat, b, torch.empty(max(pnnz, 1) * b * b, dtype=torch.float64,
                                                  device=dev))
        if pnnz:
            check(D.lib().b2s_gather_blocks(pnnz, b, D.ptr(self._own_idx),
                                            D.ptr(self.obsr.vals), D.ptr(self.pbsr.vals),
                                            D.stream()), "gather_blocks")
        # ghost couplings of the boundary rows as CSR over ghost indices (the
        # fused 2-colour loop adds them after the halo pull; b2s_mesh bnd_*)
        ub, cnt = torch.unique(rows[gh], return_counts=True)
        self._bnd_in = ub.to(torch.int64)
        bp = torch.zeros(ub.numel() + 1, dtype=torch.int64, device=dev)
        bp[1:] = torch.cumsum(cnt, 0)
        self._bnd_ptr = bp.to(torch.int32)
        ngh = int(nnz - pnnz)
        self._bnd_col = ((lcol[gh] - R).to(torch.int32) if ngh else D.empty_i32(1, dev))
        self._gh_idx = (torch.nonzero(gh).flatten().to(torch.int32) if ngh else
                        D.empty_i32(1, dev))
        self._bnd_val = torch.empty(max(ngh, 1) * b * b, dtype=torch.float64, device=dev)
        self._ngh = ngh
        self._gather_ghost_blocks()
        self.dev = dev
        if backend is not None:
            self.setup(backend)

    def setup(self, backend: Backend):
        R, dev = self.R, self.dev
        self.plan = plan_device(backend, self.pbsr.pat)
        self.fact = factor_device(self.pmat, self.plan, self.pbsr)
        # operator rows in plan order; own columns through perm, ghosts appended
        perm = self.plan.device("permutation")
        iperm = self.plan.device("inverse_permutation")
        cmap = torch.cat([perm, torch.arange(R, R + self.G, dtype=torch.int32, device=dev)])
        self._cmap, self._iperm = cmap, iperm
        self._sell = None     # whole operator (ghost columns): built on first use
        self.smap = self.fact.smap
        self._bnd_row = perm.index_select(0, self._bnd_in)
        if getattr(self, "_requests", None) is not None:
            self.set_send(self._requests)
        return self

    @property
    def sell(self) -> "D.Sell":
        """The whole operator in plan order with the ghost columns appended, as
        a SELL layout filled straight from the unpermuted values through the
        permutation's source map.  Built on first use: the fused 2-colour
        device loop never needs it (local block + ghost correction)."""
        if self._sell is None:
            opat, src = D.permute_pattern(self.obsr.pat, self._cmap, self._iperm)
            self._sell = D.Sell.build(self.smap, D.DevBSR(opat, self.b, self.obsr.vals), 0,
                                      src=src)
        return self._sell

    def _gather_ghost_blocks(self):
        nk = self._ngh
        if nk:
            check(D.lib().b2s_gather_blocks(nk, self.b, D.ptr(self._gh_idx), D.ptr(self.obsr.vals),
                                            D.ptr(self._bnd_val), D.stream()), "gather_blocks")

    def refresh_values(self, vals: np.ndarray, rhs: np.ndarray):
        """A new system with this shard's sparsity pattern (the next Newton
        step): H2D of the slab's block values and right-hand side only (async
        from page-locked buffers); the preconditioner's blocks (the owned
        columns) are gathered on the device -- the host-side halo and pattern
        work of the constructor is not repeated."""
        dev, b = self.dev, self.b
        src = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64).reshape(-1))
        self.obsr.vals.copy_(src, non_blocking=D.is_pinned(src))
        nk = self._own_idx.numel()
        check(D.lib().b2s_gather_blocks(nk, b, D.ptr(self._own_idx), D.ptr(self.obsr.vals),
                                        D.ptr(self.pbsr.vals), D.stream()), "gather_blocks")
        self._gather_ghost_blocks()
        r = torch.from_numpy(np.ascontiguousarray(rhs, dtype=np.float64))
        if getattr(self, "rhs_d", None) is None:
            self.rhs_d = torch.empty(r.numel(), dtype=torch.float64, device=dev)
        self.rhs_d.copy_(r, non_blocking=D.is_pinned(r))

    # rows this shard must send to rank h (plan-order local ids), given the
    # ghost ids rank h requested from us (gathered through the device
    # permutation: the plan never comes back to the host)
    def set_send(self, requests: dict[int, np.ndarray]):
        self._requests = requests
        if getattr(self, "_req_idx", None) is None:
            self._req_idx = {h: torch.as_tensor(np.asarray(g, dtype=np.int64) - self.slab.r0,
                                                device=self.dev)
                             for h, g in requests.items()}
        if getattr(self, "plan", None) is None:
            return               # no plan yet: setup() fills the lists
        perm = self.plan.device("permutation")
        self.send = {h: perm.index_select(0, idx) for h, idx in self._req_idx.items()}

    def vec(self, with_ghosts=False):
        return torch.zeros((self.R + (self.G if with_ghosts else 0)) * self.b,
                           dtype=torch.float64, device=self.dev)


# ---------------------------------------------------------------------------
# communicators

class LocalComm:
    """All shards in this process (one GPU): halos are device copies."""

    def __init__(self, shards):
        self.shards = shards

    def allreduce(self, vals):   # vals: per shard, 1-D CUDA tensor -> host floats
        tot = None
        for v in vals:
            h = v.cpu().numpy().astype(np.float64)
            tot = h if tot is None else tot + h
        return [tot for _ in vals]

    def halo(self, bufs):
        by_rank = {s.slab.rank: (s, x) for s, x in zip(self.shards, bufs)}
        for s, x in zip(self.shards, bufs):
            for h, idx in s.recv.items():
                src, xs = by_rank[h]
                rows = src.send[s.slab.rank]
                vals = D.gather_rows(xs, rows, len(idx), s.b)
                dst = x.view(-1, s.b)
                dst[s.R + torch.as_tensor(idx, device=x.device)] = vals.view(-1, s.b)


class NcclComm:
    """One shard per process over torch.distributed (NCCL over NVLink).  With
    a non-NCCL group (gloo: tests run two ranks on one GPU, which NCCL
    refuses) the buffers are staged through host memory."""

    def __init__(self, shard):
        import torch.distributed as dist
        self.dist = dist
        self.shards = [shard]
        self.host = dist.get_backend() != "nccl"
        s = shard
        # contiguous receive ranges per neighbour (ghost ids are sorted and
        # every owner's ids are contiguous)
        self.recv_rng = {h: (int(idx[0]), int(idx[-1]) + 1) for h, idx in s.recv.items()}

    def allreduce(self, vals):
        v = vals[0].detach().clone()
        if self.host:
            v = v.cpu()
        self.dist.all_reduce(v)
        return [v.cpu().numpy()]

    def halo(self, bufs):
        s, x = self.shards[0], bufs[0]
        ops, keep, back = [], [], []
        for h, rows in s.send.items():
            sb = D.gather_rows(x, rows, rows.numel(), s.b)
            if self.host:
                sb = sb.cpu()
            keep.append(sb)
            ops.append(self.dist.P2POp(self.dist.isend, sb, h))
        for h, (lo, hi) in self.recv_rng.items():
            rv = x[(s.R + lo) * s.b:(s.R + hi) * s.b]
            if self.host:
                staged = torch.empty(rv.numel(), dtype=rv.dtype)
                back.append((rv, staged))
                rv = staged
            ops.append(self.dist.P2POp(self.dist.irecv, rv, h))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for dst, staged in back:
            dst.copy_(staged)


def route_requests(mine, gather):
    """Tell every owner which of its rows each local slab needs.

    mine: [(rank, {owner: global ids needed})] for the slabs of this process;
    gather: all_gather_object-like callable returning everyone's lists.
    Returns {rank: {requester: global ids to send}} for the local ranks."""
    everyone = gather(mine)
    flat = [item for part in everyone for item in (part if isinstance(part, list) else [part])]
    out = {}
    for rank, _ in mine:
        out[rank] = {req: needs[rank] for req, needs in flat if rank in needs}
    return out


def exchange_requests(shards, world, gather):
    mine = [(s.slab.rank, s.halo_plan.requests()) for s in shards]
    sends = route_requests(mine, gather)
    for s in shards:
        s.set_send(sends[s.slab.rank])


# ---------------------------------------------------------------------------
# the distributed BiCGStab (bs/krylov.py:140-244 control flow)

def bicgstab_sharded(shards, comm, stop: StoppingCriteria):
    """Solve for every shard's rhs/x0 (plan order) set in ``shard.rhs_p`` /
    ``shard.x_p``; returns (report, x per shard in plan order)."""
    lib = D.lib()
    st = D.stream()
    NP = D.NPARTS
    for s in shards:
        s.scr = torch.zeros(32, dtype=torch.float64, device=s.dev)
        s.parts = torch.zeros(4 * NP, dtype=torch.float64, device=s.dev)
        s.sums = torch.zeros(4, dtype=torch.float64, device=s.dev)
        s.r = s.vec(); s.rhat = s.vec(); s.p = s.vec(); s.v = s.vec()
        s.s = s.vec(); s.t = s.vec()
        s.phat = s.vec(True); s.shat = s.vec(True); s.xg = s.vec(True)
        s.y = s.vec()
        s.xg[: s.R * s.b] = s.x_p

    def reduce(idx_list):
        """sum the partial arrays `idx_list` of every shard, then all-reduce"""
        vals = []
        for s in shards:
            for j, k in enumerate(idx_list):
                check(lib.b2s_reduce(D.ptr(s.parts[k * NP:(k + 1) * NP]), NP,
                                     D.ptr(s.sums[j:j + 1]), st), "reduce")
            vals.append(s.sums[: len(idx_list)])
        return comm.allreduce(vals)[0]

    def spmv(s, x_ext, y, mode, w, k0, k1=None):
        D.spmv(s.smap, s.sell, s.b, x_ext, y, mode, w,
               s.parts[k0 * NP:(k0 + 1) * NP],
               None if k1 is None else s.parts[k1 * NP:(k1 + 1) * NP])

    def apply_m(s, src, dst_ext):
        s.fact.apply_device(src, dst_ext)

    t0 = time.perf_counter()
    comm.halo([s.xg for s in shards])
    for s in shards:
        spmv(s, s.xg, s.r, 3, s.rhs_p, 0)
    rr0 = float(reduce([0])[0])
    n0 = float(np.sqrt(rr0))
    target = stop.relative_reduction * n0
    groups = shards[0].plan.group_count
    x0 = [s.xg[: s.R * s.b].clone() for s in shards]

    def done(conv, its, final, reason=None):
        rep = SolveReport(conv, its, n0, final, time.perf_counter() - t0, groups,
                          failure_reason=reason)
        return rep, [s.xg[: s.R * s.b] for s in shards]

    if not np.isfinite(n0):
        for s, x in zip(shards, x0):
            s.xg[: s.R * s.b] = x
        return done(False, 0.0, n0, "numerical")
    if n0 <= target or n0 == 0.0:
        return done(True, 0.0, n0)
    for s in shards:
        s.rhat.copy_(s.r)
    rho_prev = alpha = omega = 1.0
    its = 0.0
    reason = "budget"
    m = [s.R * s.b for s in shards]
    rho = rr0
    rho_known = True  # rho_0 = rhat.r = |r0|^2 (the same sum)
    for k in range(stop.max_iterations):
        if not rho_known:
            rho = float(reduce([1])[0])
        rho_known = False
        if abs(rho) < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        beta = 0.0 if k == 0 else (rho / rho_prev) * (alpha / omega)
        for s, mm in zip(shards, m):
            check(lib.b2s_vec_p(mm, k, beta, omega, D.ptr(s.r), D.ptr(s.v), D.ptr(s.p),
                                D.ptr(s.scr), st), "vec_p")
            apply_m(s, s.p, s.phat)
        comm.halo([s.phat for s in shards])
        for s in shards:
            spmv(s, s.phat, s.v, 1, s.rhat, 2)
        gamma = float(reduce([2])[0])
        if abs(gamma) < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        alpha = rho / gamma
        for s, mm in zip(shards, m):
            check(lib.b2s_vec_s(mm, alpha, D.ptr(s.r), D.ptr(s.v), D.ptr(s.phat), D.ptr(s.xg),
                                D.ptr(s.s), D.ptr(s.parts[0:NP]), NP, 0, D.ptr(s.scr), st),
                  "vec_s")
        its += 0.5
        ns = float(np.sqrt(reduce([0])[0]))
        if not np.isfinite(ns):
            reason = "numerical"
            break
        if ns <= target:
            return done(True, its, ns)
        for s in shards:
            apply_m(s, s.s, s.shat)
        comm.halo([s.shat for s in shards])
        for s in shards:
            spmv(s, s.shat, s.t, 2, s.s, 2, 3)
        tt, ts = (float(v) for v in reduce([2, 3]))
        if tt < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        omega = ts / tt
        if abs(omega) < _BREAKDOWN_FLOOR:
            reason = "breakdown"
            break
        for s, mm in zip(shards, m):
            check(lib.b2s_vec_r(mm, omega, D.ptr(s.shat), D.ptr(s.t), D.ptr(s.s),
                                D.ptr(s.rhat), D.ptr(s.xg), D.ptr(s.r), D.ptr(s.parts[0:NP]),
                                D.ptr(s.parts[NP:2 * NP]), NP, 0, D.ptr(s.scr), st), "vec_r")
        its += 0.5
        nr_rho = reduce([0, 1])
        nr = float(np.sqrt(nr_rho[0]))
        rho_next = float(nr_rho[1])
        if not np.isfinite(nr):
            reason = "numerical"
            break
        if nr <= target:
            return done(True, its, nr)
        rho_prev = rho
        rho, rho_known = rho_next, True
    comm.halo([s.xg for s in shards])
    for s in shards:
        spmv(s, s.xg, s.t, 3, s.rhs_p, 0)
    final = float(np.sqrt(reduce([0])[0]))
    finite = all(bool(torch.isfinite(s.xg[: s.R * s.b]).all()) for s in shards)
    if not finite:
        for s, x in zip(shards, x0):
            s.xg[: s.R * s.b] = x
    return done(False, its, final, reason)


def solve_shards(shards, comm, stop: StoppingCriteria, x0=None):
    """Global solve over prepared shards: rhs (input order) per shard in
    ``shard.slab.rhs``; returns (report, list of per-shard x in input order)."""
    for i, s in enumerate(shards):
        iperm = s.plan.device("inverse_permutation")
        rhs = getattr(s, "rhs_d", None)      # resident (refresh_values / an earlier solve)
        if rhs is None:
            rhs = s.rhs_d = D.f64(s.slab.rhs, s.dev)
        s.rhs_p = D.gather_rows(rhs, iperm, s.R, s.b)
        x = D.f64(x0[i], s.dev) if x0 is not None else torch.zeros_like(rhs)
        s.x_p = D.gather_rows(x, iperm, s.R, s.b)
    rep, xs = bicgstab_sharded(shards, comm, stop)
    out = []
    for s, xp in zip(shards, xs):
        out.append(D.gather_rows(xp, s.plan.device("permutation"), s.R, s.b))
    return rep, out


def local_solver(spec: GeneratorSpec, world: int, backend=Backend.LEVEL_SCHEDULED):
    """All `world` slabs of spec in this process (testing on one GPU)."""
    slabs = [generate_slab(spec, r, world) for r in range(world)]
    owners = np.array([s.r0 for s in slabs], dtype=np.int64)
    shards = [Shard(s, owners, backend) for s in slabs]
    exchange_requests(shards, world, lambda mine: [mine])
    return shards, LocalComm(shards)


def nccl_solver(spec: GeneratorSpec, backend=Backend.LEVEL_SCHEDULED):
    """This process's slab of spec (torch.distributed must be initialised)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    slab = generate_slab(spec, rank, world)
    owners = np.array([slab_bounds(spec.nz, world, r)[0] * spec.nx * spec.ny
                       for r in range(world)], dtype=np.int64)
    shard = Shard(slab, owners, backend)

    def gather(mine):
        out = [None] * world
        dist.all_gather_object(out, mine)
        return out
    exchange_requests([shard], world, gather)
    return [shard], NcclComm(shard)


# ---------------------------------------------------------------------------
# peer-memory solver: the device-resident BiCGStab loop of the single-GPU
# path (b2s_bicgstab, one CUDA graph per iteration) on every shard, with the
# communication done by the kernels themselves (csrc/krylov.cu, b2s_mesh):
# ghost rows are read straight out of the owning shard's vector, and the
# partial dot products are all-reduced through per-rank mailboxes in the
# last CTA of each reducing kernel.  No host round trip per iteration.  The
# peers are other processes' buffers opened through CUDA IPC (NVLink P2P on
# one node), or other shards on the same GPU (tests) -- the kernels are the
# same either way.

class MeshUnavailable(RuntimeError):
    """CUDA IPC / peer access between the ranks' GPUs failed on some rank
    (raised on every rank alike; the NCCL host loop still works)."""


class MeshState:
    """Device buffers of one shard for ``b2s_bicgstab`` with a ``b2s_mesh``."""

    def __init__(self, shard: "Shard", nranks: int):
        lib = D.lib()
        R, G, b, dev = shard.R, shard.G, shard.b, shard.dev
        nbytes = int(lib.b2s_bicgstab_workspace_bytes_mesh(R, G, b, D.NPARTS))
        self.work = torch.zeros(nbytes // 8 + 1, dtype=torch.float64, device=dev)
        self.x = torch.zeros((R + G) * b + 2, dtype=torch.float64, device=dev)
        self.flags = torch.zeros(max(nranks, 1), dtype=torch.int64, device=dev)
        self.mbox = torch.zeros(int(lib.b2s_mesh_mbox_bytes(nranks)) // 8, dtype=torch.float64,
                                device=dev)
        po, so = C.c_longlong(0), C.c_longlong(0)
        check(lib.b2s_bicgstab_workspace_layout(R, G, b, C.byref(po), C.byref(so)), "layout")
        self.phat = self.work.data_ptr() + 8 * po.value
        self.shat = self.work.data_ptr() + 8 * so.value
        self.nranks = nranks
        self.solves = 0
        self.peers = None         # per rank: [x, phat, shat, flags, mbox] addresses here
        self.opened = []          # IPC bases to close

    def local_ptrs(self):
        return [self.x.data_ptr(), self.phat, self.shat, self.flags.data_ptr(),
                self.mbox.data_ptr()]

    def close(self):
        for base in self.opened:
            D.lib().b2s_ipc_close(C.c_void_p(base))
        self.opened = []


def _mesh_struct(shard: "Shard", ms: MeshState, owner_rows: dict, shared_device: bool):
    """The ``_lib.Mesh`` of one shard (and the device arrays it points to)."""
    from ._lib import Mesh
    dev = shard.dev
    G = shard.G
    owner = np.zeros(max(G, 1), dtype=np.int32)
    row = np.zeros(max(G, 1), dtype=np.int32)
    for h, idx in shard.recv.items():
        owner[idx] = h
        row[idx] = np.asarray(owner_rows[h], dtype=np.int32)
    nbr = np.array(sorted(shard.recv) or [0], dtype=np.int32)
    keep = {"owner": torch.from_numpy(owner).to(dev), "row": torch.from_numpy(row).to(dev),
            "nbr": torch.from_numpy(nbr).to(dev)}
    for k, name in enumerate(("x", "phat", "shat", "flags", "mbox")):
        keep[name] = torch.tensor([p[k] for p in ms.peers], dtype=torch.int64, device=dev)
    m = Mesh()
    m.rank, m.nranks, m.nghost = shard.slab.rank, ms.nranks, G
    m.ghost_owner, m.ghost_row = D.ptr(keep["owner"]), D.ptr(keep["row"])
    m.nnbr, m.nbr = len(shard.recv), D.ptr(keep["nbr"])
    m.peer_x, m.peer_phat, m.peer_shat = (D.ptr(keep["x"]), D.ptr(keep["phat"]),
                                          D.ptr(keep["shat"]))
    m.flags, m.peer_flags = ms.flags.data_ptr(), D.ptr(keep["flags"])
    m.mbox, m.peer_mbox = ms.mbox.data_ptr(), D.ptr(keep["mbox"])
    ms.solves += 1
    m.seq_base = ms.solves << 32          # equal on every rank: one per global solve
    m.shared_device = 1 if shared_device else 0
    if _mesh_fused(shard):
        m.nbnd = int(shard._bnd_in.numel())
        m.bnd_row, m.bnd_ptr = D.ptr(shard._bnd_row), D.ptr(shard._bnd_ptr)
        m.bnd_col, m.bnd_val = D.ptr(shard._bnd_col), D.ptr(shard._bnd_val)
        # (full_*: left null -- residuals use the local block + ghost correction)
    return m, keep


def _mesh_fused(shard) -> bool:
    """2-colour shard: the fused colour passes run on the local block (the
    factorisation's own operator layout) plus the ghost correction."""
    f = shard.fact
    return (f.a_sell is not None and f.phased and not f.tiles and
            os.environ.get("B2S_FUSE", "1") != "0")


def _mesh_krylov(shard, ms):
    from .krylov import DeviceKrylov
    if _mesh_fused(shard):
        return DeviceKrylov(shard.R, shard.b, shard.smap, shard.fact.a_sell, shard.fact, ms.work,
                            True)
    return DeviceKrylov(shard.R, shard.b, shard.smap, shard.sell, shard.fact, ms.work, False)


def _mesh_prepare(shard: "Shard", nranks: int, x0=None):
    """Plan-order rhs and x0 of a shard (x0 into the mesh x buffer)."""
    if getattr(shard, "mesh", None) is None or shard.mesh.nranks != nranks or \
            shard.mesh.x.numel() != (shard.R + shard.G) * shard.b + 2:
        shard.mesh = MeshState(shard, nranks)
    ms = shard.mesh
    ms.mbox[-8:].zero_()   # the abort word (csrc/ctl.cuh abort_word): a fresh solve
    iperm = shard.plan.device("inverse_permutation")
    # the right-hand side is resident like the matrix (uploaded once per shard)
    rhs = getattr(shard, "rhs_d", None)
    if rhs is None:
        rhs = shard.rhs_d = D.f64(shard.slab.rhs, shard.dev)
    shard.rhs_p = D.gather_rows(rhs, iperm, shard.R, shard.b)
    x = D.f64(x0, shard.dev) if x0 is not None else torch.zeros_like(rhs)
    ms.x.zero_()
    ms.x[: shard.R * shard.b] = D.gather_rows(x, iperm, shard.R, shard.b)
    return ms


def _mesh_report(res, t0, groups) -> SolveReport:
    from .bridge import _report
    return _report(res, time.perf_counter() - t0, groups)


def _mesh_outputs(shards):
    return [D.gather_rows(s.mesh.x[: s.R * s.b], s.plan.device("permutation"), s.R, s.b)
            for s in shards]


def solve_shards_mesh(shards, stop: StoppingCriteria, x0=None):
    """All shards of this process on one GPU, each running the device loop on
    its own stream and host thread, communicating through peer memory.
    Returns (report, per-shard x in input order) like ``solve_shards``.
    The shards' kernels wait for each other, so every shard's stream needs its
    own hardware work queue: run with CUDA_DEVICE_MAX_CONNECTIONS >= shards + a
    few (tests/conftest.py sets 32)."""
    import threading

    N = len(shards)
    need = N + 2
    have = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
    if N > 1 and have < need:
        # shards' kernels wait for each other: a waiting kernel sharing a
        # hardware queue with its peer's would block it (until the mesh timeout)
        raise RuntimeError(f"solve_shards_mesh: {N} shards on one GPU need "
                           f"CUDA_DEVICE_MAX_CONNECTIONS >= {need} set before CUDA starts "
                           f"(it is {have})")
    by_rank = {s.slab.rank: s for s in shards}
    mss = [_mesh_prepare(s, N, None if x0 is None else x0[i]) for i, s in enumerate(shards)]
    ptrs = [by_rank[r].mesh.local_ptrs() for r in range(N)]
    # the shards' host threads rendezvous around the device loop (b2s_mesh
    # host_barrier): on one GPU, no shard may make an implicitly
    # synchronising call while another shard's kernel waits for it
    from ._lib import BARRIER_FN
    rendezvous = threading.Barrier(N)

    def _barrier(_ctx):   # ctypes swallows exceptions: report failure as a status
        try:
            rendezvous.wait()
            return 0
        except threading.BrokenBarrierError:
            return 1
    barrier_cb = BARRIER_FN(_barrier)
    jobs = []
    for s, ms in zip(shards, mss):
        ms.peers = ptrs
        me = s.slab.rank
        owner_rows = {h: by_rank[h].send[me].cpu().numpy() for h in s.recv}
        mesh, keep = _mesh_struct(s, ms, owner_rows, shared_device=True)
        mesh.host_barrier = C.cast(barrier_cb, C.c_void_p)
        keep["barrier"] = barrier_cb
        kr = _mesh_krylov(s, ms)
        jobs.append((s, ms, kr, mesh, keep))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    results, errors = [None] * N, []

    def run(i):
        s, ms, kr, mesh, _ = jobs[i]
        try:
            st = getattr(s, "_mesh_stream", None)
            if st is None:   # one persistent stream per shard (see b2s_mesh shared_device)
                st = s._mesh_stream = torch.cuda.Stream(device=s.dev)
            with torch.cuda.stream(st):
                results[i] = kr.solve(s.rhs_p, ms.x, stop, mesh=mesh, x0_zero=x0 is None)
                st.synchronize()
        except Exception as exc:   # surfaced below, after every thread is back
            errors.append(exc)
            rendezvous.abort()
    threads = [threading.Thread(target=run, args=(i,)) for i in range(N)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    if errors:
        raise errors[0]
    rep = _mesh_report(results[0], t0, shards[0].plan.group_count)
    for r in results[1:]:
        assert r.iterations == results[0].iterations and r.converged == results[0].converged
    return rep, _mesh_outputs(shards)


def solve_shard_mesh_dist(shard: "Shard", stop: StoppingCriteria, x0=None, cache_key=None):
    """This process's shard of a torch.distributed job (one GPU per rank):
    peers' buffers are opened once through CUDA IPC (NVLink P2P)."""
    import torch.distributed as dist

    from .krylov import DeviceKrylov
    rank, world = dist.get_rank(), dist.get_world_size()
    tm = [time.perf_counter()]
    dist.barrier()       # every peer is done reading this rank's x of the last solve
    tm.append(time.perf_counter())
    ms = _mesh_prepare(shard, world, x0)

    def gather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out
    lib = D.lib()
    if ms.peers is None:
        # every rank exports its buffers and opens every peer's; a failure on
        # any rank (no IPC / peer access between these GPUs) is agreed on by
        # all of them before anyone waits on a peer, and raised everywhere as
        # MeshUnavailable -- the caller can fall back to the NCCL host loop
        err = None
        mine = []
        try:
            for p in ms.local_ptrs():
                h = (C.c_ubyte * 64)()
                off = C.c_longlong(0)
                check(lib.b2s_ipc_handle(C.c_void_p(p), h, C.byref(off)), "ipc_handle")
                mine.append((bytes(h), off.value))
        except Exception as exc:
            err = repr(exc)
        peers = [None] * world
        for r, hs in gather((rank, mine if err is None else None)):
            if r == rank:
                peers[r] = ms.local_ptrs()
                continue
            opened = []
            try:
                if err is None and hs is not None:
                    for hb, off in hs:
                        out = C.c_void_p(None)
                        buf = (C.c_ubyte * 64).from_buffer_copy(hb)
                        check(lib.b2s_ipc_open(buf, off, C.byref(out)), "ipc_open")
                        opened.append(out.value)
                        ms.opened.append(out.value - off)
            except Exception as exc:
                err = repr(exc)
            peers[r] = opened
        verdicts = gather((rank, err))
        bad = [(r, e) for r, e in verdicts if e is not None]
        if bad or any(h is None for h in peers):
            ms.close()
            raise MeshUnavailable("; ".join(f"rank {r}: {e}" for r, e in bad)
                                  or "a peer could not export its buffers")
        ms.peers = peers
    key = ("owner_rows", cache_key)
    if getattr(shard, "_owner_rows_key", None) != key:
        sends = {h: rows.cpu().numpy() for h, rows in shard.send.items()}
        everyone = gather((rank, sends))
        shard._owner_rows = {r: d[rank] for r, d in everyone if rank in d}
        shard._owner_rows_key = key
    mesh, keep = _mesh_struct(shard, ms, shard._owner_rows, shared_device=False)
    kr = _mesh_krylov(shard, ms)
    t0 = time.perf_counter()
    tm.append(t0)
    res = kr.solve(shard.rhs_p, ms.x, stop, mesh=mesh, x0_zero=x0 is None)
    tm.append(time.perf_counter())
    rep = _mesh_report(res, t0, shard.plan.group_count)
    out = _mesh_outputs([shard])[0]
    if os.environ.get("B2S_MESH_TIMING") == "1":
        torch.cuda.synchronize()
        tm.append(time.perf_counter())
        print("mesh timing ms (barrier, prepare, solve, outputs):",
              [round((b - a) * 1e3, 3) for a, b in zip(tm, tm[1:])], flush=True)
    return rep, out
