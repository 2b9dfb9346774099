"""Device mirrors of the reference's data types and the thin engine layer.

Host objects (``BlockMatrix``/``BlockVector``/``ParallelPlan``) keep the
reference's numpy-facing API; everything numeric happens on the GPU through
libb200solve.so.  Device buffers are torch CUDA tensors owned by Python (the
C side only receives pointers, sizes and the current stream).

Layout in HBM:
  * pattern: int32 row pointers (n+1) and column indices (nnzb);
  * values: fp64 canonical block-row-major (nnzb*b*b);
  * block vectors: fp64 interleaved [row][b];
  * SELL-32 tiles built once per matrix for the bandwidth-bound kernels.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check

NPARTS = 148 * 4   # CTAs of every reducing kernel: fixed => deterministic sums

_I32_MAX = 2 ** 31 - 1


_configured = set()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2309_11488_b200 needs a CUDA device (no CPU fallback)")
    d = torch.cuda.current_device()
    if d not in _configured:
        check(lib().b2s_retain_pool_memory(d), "retain_pool_memory")
        _configured.add(d)
    return torch.device("cuda", d)


def lib():
    return _lib.load()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def i32(a: np.ndarray, dev) -> torch.Tensor:
    """int32 device copy of an index array.  Large int64 arrays travel as they
    are and are narrowed (and range-checked) by a device kernel."""
    a = np.asarray(a)
    if a.dtype == np.int64 and a.size >= (1 << 16):
        src = torch.from_numpy(np.ascontiguousarray(a))
        raw = to_device(src, dev)
        out = torch.empty(a.size, dtype=torch.int32, device=dev)
        bad = C.c_int(0)
        check(lib().b2s_narrow_index(a.size, ptr(raw), ptr(out), C.byref(bad), stream()),
              "narrow_index")
        if bad.value:
            raise ValueError("index does not fit the device's int32 indices")
        return out
    if a.size and (a.max() > _I32_MAX or a.min() < -_I32_MAX):
        raise ValueError("index does not fit the device's int32 indices")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev, non_blocking=False)


def f64(a: np.ndarray, dev) -> torch.Tensor:
    src = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    return to_device(src, dev)


_UPLOAD: dict = {}


def upload_stream(dev) -> torch.cuda.Stream:
    """The device's copy stream for overlapped uploads, one per process.  (A
    new stream per call leaked a caching-allocator segment per solve: blocks
    allocated on a stream are only reused by that stream -- measured +23 MB
    reserved and one cudaMalloc per C4 solve, tools/e2e_phases.py.)"""
    dev = torch.device(dev)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    st = _UPLOAD.get(idx)
    if st is None:
        st = _UPLOAD[idx] = torch.cuda.Stream(device=dev)
    return st


def to_device(src: torch.Tensor, dev, stream=None) -> torch.Tensor:
    """Host tensor -> new device tensor: plain async DMA from page-locked
    memory, the staged path (staged_copy) for large pageable arrays."""
    if is_pinned(src) or src.numel() * src.element_size() < STAGE_MIN_BYTES:
        if stream is None:
            return src.to(dev, non_blocking=is_pinned(src))
        with torch.cuda.stream(stream):
            return src.to(dev, non_blocking=is_pinned(src))
    out = torch.empty(src.shape, dtype=src.dtype, device=dev)
    staged_copy(out, src, stream or torch.cuda.current_stream(dev))
    return out


# ---------------------------------------------------------------------------
# pageable host -> device at DMA speed.  A copy out of ordinary (pageable)
# numpy memory goes through the driver's own staging at a fraction of the
# PCIe rate; here chunks are memcpy'd by a few host threads into a ring of
# page-locked buffers and DMA'd from there while the next chunks are copied.

STAGE_CHUNK = int(os.environ.get("B2S_STAGE_CHUNK_MB", "8")) << 20
STAGE_BUFS = int(os.environ.get("B2S_STAGE_BUFS", "8"))
STAGE_MIN_BYTES = 4 << 20
_STAGERS: dict = {}


class _Stager:
    def __init__(self, dev):
        import concurrent.futures as cf
        import threading
        self.bufs = [torch.empty(STAGE_CHUNK, dtype=torch.uint8, pin_memory=True)
                     for _ in range(STAGE_BUFS)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * STAGE_BUFS     # last DMA out of each buffer
        workers = int(os.environ.get("B2S_STAGE_THREADS", "0")) or \
            min(STAGE_BUFS - 1, max(2, (os.cpu_count() or 4) // 2))
        self.workers = workers
        self.pool = cf.ThreadPoolExecutor(max_workers=workers)
        self.lock = threading.Lock()


def staged_copy(dst: torch.Tensor, src: torch.Tensor, stream) -> None:
    """dst (contiguous device tensor) <- src (contiguous pageable host tensor of
    the same byte size; or int64 -> int32, narrowed while staging -- the
    caller guarantees the values fit), DMAs enqueued on ``stream``; returns
    once every chunk is in flight (the ring's buffers are reused only after
    their DMA)."""
    narrow = src.dtype == torch.int64 and dst.dtype == torch.int32
    if narrow:
        nbytes = src.numel()            # (counted in destination elements)
        esz = 4
    else:
        nbytes = src.numel() * src.element_size()
        esz = 1
    if nbytes == 0:
        return
    dev = dst.device
    st = _STAGERS.get(dev.index)
    if st is None:
        st = _STAGERS[dev.index] = _Stager(dev)
    if narrow:
        s8 = src.reshape(-1).numpy()
        d8 = dst.reshape(-1)
    else:
        s8 = src.reshape(-1).view(torch.uint8).numpy()
        d8 = dst.reshape(-1).view(torch.uint8)
    # arrays of a few chunks are cut finer so every copy thread gets a share
    # (an 8 MB array would otherwise be one thread's memcpy)
    chunk = min(STAGE_CHUNK // esz, max((1 << 20) // esz, -(-nbytes // st.workers)))
    chunk = -(-chunk // 4096) * 4096
    nch = (nbytes + chunk - 1) // chunk
    with st.lock:
        def fill(i):
            b = i % STAGE_BUFS
            ev = st.events[b]
            if ev is not None:
                ev.synchronize()
            lo = i * chunk
            hi = min(nbytes, lo + chunk)
            if narrow:
                np.copyto(st.views[b].view(np.int32)[: hi - lo], s8[lo:hi], casting="unsafe")
            else:
                np.copyto(st.views[b][: hi - lo], s8[lo:hi])
        futs = {}
        for i in range(min(STAGE_BUFS - 1, nch)):
            futs[i] = st.pool.submit(fill, i)
        for i in range(nch):
            futs.pop(i).result()
            b = i % STAGE_BUFS
            lo = i * chunk
            hi = min(nbytes, lo + chunk)
            with torch.cuda.stream(stream):
                buf = st.bufs[b].view(torch.int32) if narrow else st.bufs[b]
                d8[lo:hi].copy_(buf[: hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(stream)
            st.events[b] = ev
            if i + STAGE_BUFS - 1 < nch:
                futs[i + STAGE_BUFS - 1] = st.pool.submit(fill, i + STAGE_BUFS - 1)


def is_pinned(t: torch.Tensor) -> bool:
    """Page-locked host memory (cudaHostAlloc / torch pin_memory): copies from
    it are plain DMA and can run asynchronously."""
    try:
        return bool(t.numel()) and t.is_pinned()
    except RuntimeError:
        return False


def pinned_empty(n: int, dtype=np.float64) -> np.ndarray:
    """A numpy array backed by page-locked host memory (torch's caching host
    allocator: freed arrays go back to a pool, so repeated solves reuse them)."""
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.int64): torch.int64,
           np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
    return torch.empty(int(n), dtype=tdt, pin_memory=True).numpy()


def pinned_copy(a: np.ndarray) -> np.ndarray:
    out = pinned_empty(np.asarray(a).size, np.asarray(a).dtype)
    out[:] = np.asarray(a).reshape(-1)
    return out.reshape(np.shape(a))


def pin_host(obj):
    """Copy of a BlockMatrix / BlockVector (or array) whose arrays live in
    page-locked host memory -- what an assembler hands the solver when the
    upload should run at DMA speed."""
    from .blockcore import BlockMatrix, BlockVector, SparsityPattern
    if isinstance(obj, BlockMatrix):
        p = obj.pattern
        pat = SparsityPattern(p.num_block_rows, pinned_copy(p.row_pointers),
                              pinned_copy(p.column_indices))
        return BlockMatrix(pat, obj.block_size, pinned_copy(obj.values), obj.layout)
    if isinstance(obj, BlockVector):
        return BlockVector(pinned_copy(obj.data), obj.block_size)
    return pinned_copy(obj)


def to_host_vector(v: torch.Tensor, count: int, block_size: int):
    """The solution as a host BlockVector: finiteness is checked on the device
    (one reduction) instead of on the host, then one D2H into pinned memory."""
    from .blockcore import BlockVector
    if not all_finite(v, int(count)):
        raise ValueError("block vector entries must be finite")
    return BlockVector._checked_on_device(to_host(v, count), block_size)


class HostResult:
    """A solve's result on its way to the host: the finiteness check, the
    D2H of x into page-locked memory and any further device scalars are all
    queued first, then one synchronisation (no device idle between small
    reads)."""

    def __init__(self, v: torch.Tensor, count: int, block_size: int):
        count = int(count)
        self.count, self.block_size = count, block_size
        self._bad = torch.zeros(1, dtype=torch.int32, device=v.device)
        check(lib().b2s_all_finite(count, ptr(v), ptr(self._bad), stream()), "all_finite")
        self._bad_h = torch.empty(1, dtype=torch.int32, pin_memory=True)
        self._bad_h.copy_(self._bad, non_blocking=True)
        self._x = torch.empty(count, dtype=v.dtype, pin_memory=True)
        if count:
            self._x.copy_(v[:count], non_blocking=True)
        self._extra = []

    def fetch(self, t: torch.Tensor) -> int:
        """Queue a small device tensor's D2H; its value is ``value(k)`` after wait()."""
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        self._extra.append(h)
        return len(self._extra) - 1

    def wait(self):
        torch.cuda.current_stream().synchronize()
        return self

    def value(self, k: int) -> torch.Tensor:
        return self._extra[k]

    def vector(self):
        from .blockcore import BlockVector
        if int(self._bad_h.item()):
            raise ValueError("block vector entries must be finite")
        return BlockVector._checked_on_device(self._x.numpy(), self.block_size)


def to_host(v: torch.Tensor, count: int) -> np.ndarray:
    """D2H of the first ``count`` elements into page-locked memory (fast DMA;
    the returned array owns a pinned block of the caching host allocator)."""
    out = torch.empty(int(count), dtype=v.dtype, pin_memory=True)
    if count:
        out.copy_(v[: int(count)], non_blocking=True)
        torch.cuda.current_stream().synchronize()
    return out.numpy()


def empty_i32(n, dev):
    return torch.empty(max(int(n), 1), dtype=torch.int32, device=dev)


def empty_f64(n, dev):
    return torch.empty(max(int(n), 1), dtype=torch.float64, device=dev)


# ---------------------------------------------------------------------------

def grid_hint(n: int, rp: np.ndarray, ci: np.ndarray):
    """(nx, ny) if the couplings of the middle row look like a natural-order
    nx x ny x nz stencil (positive offsets {1, nx, nx*ny}, or a 2-D / 1-D
    subset), else None.  A hint only: the plan kernels verify any guess built
    from it against every row, so a wrong hint costs one pass, never a result."""
    if n < 8:
        return None
    best = None
    # a row on the top plane has no z+1 coupling (nz = 2: the middle row is
    # one), so a few rows are looked at and the richest reading kept
    for r in (n // 2, n // 4, (3 * n) // 4):
        off = np.asarray(ci[int(rp[r]):int(rp[r + 1])], dtype=np.int64) - r
        u = [int(v) for v in np.unique(off[off > 0])]
        if len(u) == 3 and u[0] == 1 and u[2] % u[1] == 0 and n % u[2] == 0:
            return u[1], u[2] // u[1]
        if best is None and u == [1]:
            best = (n, 1)
        elif len(u) == 2 and u[0] == 1 and n % u[1] == 0 and (best is None or best[1] == 1):
            best = (u[1], n // u[1])
    return best


@dataclass
class DevPattern:
    n: int
    nnz: int
    rp: torch.Tensor
    ci: torch.Tensor
    grid: tuple | None = None    # grid_hint of the host pattern

    @classmethod
    def upload(cls, pattern) -> "DevPattern":
        dev = require_cuda()
        n = int(pattern.num_block_rows)
        rp = np.asarray(pattern.row_pointers)
        ci = np.asarray(pattern.column_indices)
        return cls(n, int(rp[-1]) if n else 0, i32(rp, dev), i32(ci, dev) if ci.size
                   else empty_i32(1, dev), grid_hint(n, rp, ci))

    def host(self):
        rp = self.rp[: self.n + 1].cpu().numpy().astype(np.int64)
        ci = self.ci[: self.nnz].cpu().numpy().astype(np.int64)
        return rp, ci


@dataclass
class DevBSR:
    pat: DevPattern
    b: int
    vals: torch.Tensor

    @classmethod
    def upload(cls, m, overlap: bool = False) -> "DevBSR":
        """Pattern first, then the values.  With ``overlap`` every host->device
        copy runs back to back on the device's upload stream (page-locked
        arrays: plain async DMA; pageable: the staging ring, from a helper
        thread) and the caller goes on as soon as the pattern is queued: the
        indices are narrowed on the current stream behind an event and the
        pattern-only work (the analysis) overlaps the value copy;
        ``wait_values()`` orders the current stream after it."""
        m = m.as_block_row_major()
        if not overlap or not m.values.size:
            pat = DevPattern.upload(m.pattern)
            dev = pat.rp.device
            if not m.values.size:
                return cls(pat, int(m.block_size), empty_f64(1, dev))
            out = cls(pat, int(m.block_size), torch.empty(m.values.size, dtype=torch.float64,
                                                           device=dev))
            src = torch.from_numpy(m.values)
            if is_pinned(src) or src.numel() * 8 < STAGE_MIN_BYTES:
                out.vals.copy_(src, non_blocking=is_pinned(src))
            else:
                staged_copy(out.vals, src, torch.cuda.current_stream(dev))
            return out
        dev = require_cuda()
        p = m.pattern
        n = int(p.num_block_rows)
        rp_h = np.ascontiguousarray(p.row_pointers, dtype=np.int64)
        ci_h = np.ascontiguousarray(p.column_indices, dtype=np.int64)
        nnz = int(rp_h[-1]) if n else 0
        # a SparsityPattern checked 0 <= ci < n and 0 = rp[0] <= ... <= nnz at
        # construction: with n and nnz inside int32 no index can overflow, so
        # the narrowing needs no host read (DevPattern.upload keeps the check)
        if n > _I32_MAX or nnz > _I32_MAX:
            raise ValueError("index does not fit the device's int32 indices")
        cur = torch.cuda.current_stream(dev)
        side = upload_stream(dev)
        side.wait_stream(cur)
        rp_t, ci_t = torch.from_numpy(rp_h), torch.from_numpy(ci_h)
        # page-locked indices travel as they are and are narrowed on the
        # device; pageable ones are narrowed while staging (half the bytes)
        direct = is_pinned(rp_t) and (nnz == 0 or is_pinned(ci_t))
        it = torch.int64 if direct else torch.int32
        rp_raw = torch.empty(n + 1, dtype=it, device=dev)
        ci_raw = torch.empty(max(nnz, 1), dtype=it, device=dev)
        vals = torch.empty(m.values.size, dtype=torch.float64, device=dev)
        srcs = [(rp_raw, rp_t), (ci_raw[:nnz], ci_t), (vals, torch.from_numpy(m.values))]
        ev_pat, done = torch.cuda.Event(), torch.cuda.Event()
        import threading
        queued = threading.Event()

        errors: list = []

        def copy_all():
            try:
                for i, (dst, src) in enumerate(srcs):
                    if src.numel() == 0:
                        pass
                    elif dst.dtype == src.dtype and (
                            is_pinned(src) or src.numel() * src.element_size() < STAGE_MIN_BYTES):
                        with torch.cuda.stream(side):
                            dst.copy_(src, non_blocking=is_pinned(src))
                    else:
                        staged_copy(dst, src, side)
                    if i == 1:
                        ev_pat.record(side)
                        queued.set()
                done.record(side)
            except BaseException as exc:   # re-raised by the caller / wait_values
                errors.append(exc)
            finally:
                queued.set()
        if all(is_pinned(src) for _, src in srcs if src.numel()):
            copy_all()   # page-locked: every DMA is asynchronous, no helper thread
            th = None
        else:
            th = threading.Thread(target=copy_all, daemon=True)
            th.start()
            queued.wait()
        if errors:
            if th is not None:
                th.join()
            raise errors[0]
        cur.wait_event(ev_pat)
        if direct:
            rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
            ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
            check(lib().b2s_narrow_index(n + 1, ptr(rp_raw), ptr(rp), None, stream()),
                  "narrow_index")
            check(lib().b2s_narrow_index(nnz, ptr(ci_raw), ptr(ci), None, stream()),
                  "narrow_index")
        else:
            rp, ci = rp_raw, ci_raw
        pat = DevPattern(n, nnz, rp, ci, grid_hint(n, rp_h, ci_h))
        out = cls(pat, int(m.block_size), vals)
        out._pending = (th, done)
        out._side = side
        out._errors = errors
        return out

    def upload_after(self, a: np.ndarray) -> torch.Tensor:
        """fp64 device copy of ``a`` queued behind the (overlapped) value
        upload, so the current stream's pattern analysis does not wait for
        it on the copy engine; ordered by wait_values()."""
        side = getattr(self, "_side", None)
        pending = getattr(self, "_pending", None)
        src = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        if side is None or pending is None:
            return f64(a, self.vals.device)
        th, _ = pending
        done = torch.cuda.Event()
        if th is not None:   # pageable values still being staged: queue behind them
            import threading
            out = torch.empty(src.numel(), dtype=torch.float64, device=self.vals.device)

            def copy(prev=th):
                prev.join()
                staged_copy(out, src, side)
                with torch.cuda.stream(side):
                    done.record(side)
            t2 = threading.Thread(target=copy, daemon=True)
            t2.start()
            self._pending = (t2, done)
            return out
        out = to_device(src, self.vals.device, side)
        with torch.cuda.stream(side):
            done.record(side)
        self._pending = (None, done)
        return out

    def wait_values(self):
        pending = getattr(self, "_pending", None)
        if pending is not None:
            th, ev = pending
            if th is not None:
                th.join()
            self._pending = None
            errors = getattr(self, "_errors", None)
            if errors:
                raise errors[0]
            torch.cuda.current_stream().wait_event(ev)


def find_diagonal(p: DevPattern) -> torch.Tensor:
    """Diagonal slot of every row (MissingDiagonal otherwise); kept on the
    pattern, which never changes, so a later caller costs no device round trip."""
    diag = getattr(p, "_diag", None)
    if diag is not None:
        return diag
    diag = empty_i32(p.n, p.rp.device)
    bad = C.c_int32(-1)
    rc = lib().b2s_find_diagonal(p.n, ptr(p.rp), ptr(p.ci), ptr(diag), C.byref(bad), stream())
    check(rc, "find_diagonal", bad.value)
    p._diag = diag
    return diag


def groups(p: DevPattern, kind: str):
    """Device level schedule / colouring; returns (row_group int32, ngroups)."""
    g = empty_i32(p.n, p.rp.device)
    ng = C.c_int32(0)
    used = C.c_int(0)
    fn = lib().b2s_level_schedule_hint if kind == "level" else lib().b2s_graph_color_hint
    # MissingDiagonal first, exactly like bs/analysis.py:79-82
    find_diagonal(p)
    nx, ny = (p.grid if p.grid is not None and os.environ.get("B2S_PLAN_HINT", "1") != "0"
              else (0, 0))
    check(fn(p.n, ptr(p.rp), ptr(p.ci), nx, ny, ptr(g), C.byref(ng), C.byref(used), stream()),
          kind)
    p.hint_used = bool(used.value)
    return g, int(ng.value)


def plan_arrays(row_group: torch.Tensor, n: int, ngroups: int):
    dev = row_group.device
    perm = empty_i32(n, dev)
    iperm = empty_i32(n, dev)
    off = empty_i32(ngroups + 1, dev)
    check(lib().b2s_plan_from_groups(n, ptr(row_group), ngroups, ptr(perm), ptr(iperm),
                                     ptr(off), stream()), "plan_from_groups")
    return perm, iperm, off


def permute(m: DevBSR, cmap: torch.Tensor, take: torch.Tensor, want_src=False):
    p = m.pat
    dev = p.rp.device
    rp = empty_i32(p.n + 1, dev)
    ci = empty_i32(p.nnz, dev)
    bb = m.b * m.b
    vals = empty_f64(p.nnz * bb, dev)
    src = empty_i32(p.nnz, dev) if want_src else None
    check(lib().b2s_permute_bsr(p.n, m.b, ptr(p.rp), ptr(p.ci), ptr(m.vals), ptr(cmap),
                                ptr(take), ptr(rp), ptr(ci), ptr(vals), ptr(src), stream()),
          "permute_bsr")
    out = DevBSR(DevPattern(p.n, p.nnz, rp, ci), m.b, vals)
    return (out, src) if want_src else out


def permute_pattern(p: DevPattern, cmap: torch.Tensor, take: torch.Tensor):
    """Plan-order pattern and the source map (input slot of every plan-order
    slot), without moving any values."""
    dev = p.rp.device
    rp = empty_i32(p.n + 1, dev)
    ci = empty_i32(p.nnz, dev)
    src = empty_i32(p.nnz, dev)
    check(lib().b2s_permute_bsr(p.n, 1, ptr(p.rp), ptr(p.ci), None, ptr(cmap), ptr(take),
                                ptr(rp), ptr(ci), None, ptr(src), stream()), "permute_pattern")
    return DevPattern(p.n, p.nnz, rp, ci), src


def gather_rows(v: torch.Tensor, src: torch.Tensor, n: int, b: int,
                out: torch.Tensor | None = None) -> torch.Tensor:
    if out is None:
        out = torch.empty(n * b, dtype=torch.float64, device=v.device)
    check(lib().b2s_gather_rows(n, b, ptr(src), ptr(v), ptr(out), stream()), "gather_rows")
    return out


# ---------------------------------------------------------------------------
# slice maps and SELL-32 layouts

PHASED_MAX_GROUPS = 32   # plans with at most this many groups may use phased sweeps


@dataclass
class SliceMap:
    nslices: int
    row0: torch.Tensor
    nrows: torch.Tensor
    gslice_host: np.ndarray | None = None   # group g -> first slice (few-group plans)
    goff1: int = 0                          # first row of group 1

    @classmethod
    def plain(cls, n: int, dev) -> "SliceMap":
        ns = (n + 31) // 32
        row0, nrows = empty_i32(ns, dev), empty_i32(ns, dev)
        check(lib().b2s_slices_plain(n, ptr(row0), ptr(nrows), stream()), "slices_plain")
        return cls(ns, row0, nrows)

    @classmethod
    def grouped(cls, offsets: torch.Tensor, ngroups: int) -> "SliceMap":
        dev = offsets.device
        base = empty_i32(ngroups + 1, dev)
        ns = C.c_int32(0)
        check(lib().b2s_slices_grouped_count(ngroups, ptr(offsets), ptr(base), C.byref(ns),
                                             stream()), "slices_grouped")
        row0, nrows = empty_i32(ns.value, dev), empty_i32(ns.value, dev)
        check(lib().b2s_slices_grouped_fill(ngroups, ns.value, ptr(offsets), ptr(base),
                                            ptr(row0), ptr(nrows), stream()), "slices_grouped")
        out = cls(int(ns.value), row0, nrows)
        if 2 <= ngroups <= PHASED_MAX_GROUPS:
            # host copy of the group -> slice table: the phased sweeps launch
            # one pass per group (the table is baked into the captured graph)
            # (one readback for the table and the first group's size)
            both = torch.cat([base[: ngroups + 1], offsets[1:2].to(torch.int32)]).cpu().numpy()
            out.gslice_host = np.ascontiguousarray(both[: ngroups + 1], dtype=np.int32)
            out.goff1 = int(both[ngroups + 1])
        return out

    @classmethod
    def singles(cls, n: int, dev) -> "SliceMap":
        """One row per slice: always safe for the triangular sweeps."""
        row0 = torch.arange(max(n, 1), dtype=torch.int32, device=dev)
        nrows = torch.ones(max(n, 1), dtype=torch.int32, device=dev)
        return cls(n, row0, nrows)

    def conflicts(self, p: DevPattern) -> bool:
        c = C.c_int(0)
        check(lib().b2s_slice_conflicts(self.nslices, ptr(self.row0), ptr(self.nrows),
                                        ptr(p.rp), ptr(p.ci), C.byref(c), stream()),
              "slice_conflicts")
        return bool(c.value)


@dataclass
class Sell:
    sp: torch.Tensor
    cols: torch.Tensor
    vals: torch.Tensor
    slots: int
    width: int   # widest slice (entries)
    stale: bool = False  # some entry reads a same-group (pre-sweep) value

    @classmethod
    def build(cls, smap: SliceMap, m: DevBSR, sel: int, goff: torch.Tensor | None = None,
              ngroups: int = 0, src: torch.Tensor | None = None,
              fill: bool = True) -> "Sell":
        """SELL-32 copy of ``m`` (sel 0 all / 1 strict lower / 2 strict upper);
        with plan group offsets, same-group triangular entries are marked.
        ``src``: values of pattern slot q come from slot src[q] of ``m.vals``
        (a permuted layout filled from the unpermuted values).  ``fill=False``
        only sizes and allocates the layout (a kernel fills it later)."""
        dev = m.pat.rp.device
        sp = empty_i32(smap.nslices + 1, dev)
        slots = C.c_longlong(0)
        wmax = C.c_int(0)
        check(lib().b2s_sell_offsets_ex(smap.nslices, ptr(smap.row0), ptr(smap.nrows),
                                        ptr(m.pat.rp), ptr(m.pat.ci), sel, ptr(sp),
                                        C.byref(slots), C.byref(wmax), stream()), "sell_offsets")
        ns = int(slots.value)
        if ns * m.b * m.b > _I32_MAX * 8:
            raise ValueError("matrix too large for one device layout")
        cols = empty_i32(ns, dev)
        vals = empty_f64(ns * m.b * m.b, dev)
        if fill:
            check(lib().b2s_sell_fill_src(smap.nslices, m.b, ptr(smap.row0), ptr(smap.nrows),
                                          ptr(m.pat.rp), ptr(m.pat.ci), ptr(m.vals), sel,
                                          ptr(sp), ptr(goff), int(ngroups), ptr(cols),
                                          ptr(vals), ptr(src), stream()), "sell_fill")
        width = int(wmax.value)
        stale = (bool((cols[:ns] <= -2).any().item())
                 if (fill and goff is not None and ns) else False)
        return cls(sp, cols, vals, ns, width, stale)

    def fill_from(self, smap: SliceMap, m: DevBSR, sel: int, src: torch.Tensor | None = None):
        """Fill a layout sized by ``build(..., fill=False)`` (values of ``m``,
        through ``src`` when given) -- the value pass of a two-step build."""
        check(lib().b2s_sell_fill_src(smap.nslices, m.b, ptr(smap.row0), ptr(smap.nrows),
                                      ptr(m.pat.rp), ptr(m.pat.ci), ptr(m.vals), sel,
                                      ptr(self.sp), None, 0, ptr(self.cols), ptr(self.vals),
                                      ptr(src), stream()), "sell_fill")


def spmv(smap: SliceMap, a: Sell, b: int, x: torch.Tensor, y: torch.Tensor, mode: int = 0,
         w: torch.Tensor | None = None, parts0=None, parts1=None):
    check(lib().b2s_spmv(b, mode, NPARTS, smap.nslices, ptr(smap.row0), ptr(smap.nrows),
                         ptr(a.sp), ptr(a.cols), ptr(a.vals), ptr(x), ptr(y), ptr(w),
                         ptr(parts0), ptr(parts1), None, stream()), "spmv")


def dot(a: torch.Tensor, b: torch.Tensor, m: int) -> float:
    dev = a.device
    parts = torch.empty(NPARTS, dtype=torch.float64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    check(lib().b2s_dot(m, ptr(a), ptr(b), NPARTS, ptr(parts), ptr(out), stream()), "dot")
    return float(out.item())


def dot_chunked(a: torch.Tensor, b: torch.Tensor, m: int, partials: bool = False):
    """The reference's chunk-64 inner product (bs/krylov.py:30-47), bit for bit
    (csrc/refdot.cu).  Returns the device total (1 double) or, with
    ``partials``, the per-chunk partial sums."""
    dev = a.device
    np_ = (int(m) + 63) // 64
    parts = torch.empty(max(np_, 1), dtype=torch.float64, device=dev)
    out = None if partials else torch.empty(1, dtype=torch.float64, device=dev)
    check(lib().b2s_dot_chunked(int(m), ptr(a), ptr(b), ptr(parts), ptr(out), stream()),
          "dot_chunked")
    return parts[:np_] if partials else out


def fill_sentinel(v: torch.Tensor, m: int):
    check(lib().b2s_fill_sentinel(m, ptr(v), stream()), "fill_sentinel")


def all_finite(v: torch.Tensor, m: int) -> bool:
    bad = torch.zeros(1, dtype=torch.int32, device=v.device)
    check(lib().b2s_all_finite(m, ptr(v), ptr(bad), stream()), "all_finite")
    return not bool(bad.item())
