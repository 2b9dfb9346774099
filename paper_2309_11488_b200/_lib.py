"""ctypes binding of libb200solve.so (declared in include/b200solve.h).

The library is the only compute path of this package.  It is loaded from
the package directory (built in-tree by ``build.py``); if it is missing or
no CUDA device is visible, every entry point raises -- there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import MissingDiagonal, ShapeError, SingularPivot

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("B2S_LIB", _PKG / "libb200solve.so"))

OK, SHAPE, MISSING_DIAGONAL, SINGULAR_PIVOT, CUDA_ERROR, UNSUPPORTED, PEER_TIMEOUT = range(7)

_P = C.c_void_p
_I = C.c_int
_LL = C.c_longlong
_PI = C.POINTER(C.c_int32)
_PLL = C.POINTER(C.c_longlong)


class BicgArgs(C.Structure):
    _fields_ = [("n", _I), ("b", _I), ("nparts", _I), ("precond", _I), ("kc", _I),
                ("maxit", _I), ("check_lag", _I), ("refill_y", _I), ("sweep_flags", _I),
                ("tol", C.c_double), ("nslices", _I),
                ("row0", _P), ("nrows", _P), ("a_sp", _P), ("a_cols", _P), ("a_vals", _P),
                ("l_sp", _P), ("l_cols", _P), ("l_vals", _P),
                ("u_sp", _P), ("u_cols", _P), ("u_vals", _P),
                ("dinv_tiles", _P), ("tiles", _P), ("rhs", _P), ("x", _P), ("work", _P),
                ("stream", _P), ("ngroups", _I), ("goff1", _I), ("gslice_host", _P),
                ("fuse", _I), ("mesh", _P), ("x0_zero", _I),
                ("wells", _P), ("well_slice", _P), ("well_lane", _P), ("well_corr", _P),
                ("well_scratch", _P), ("gw", _P)]


class Mesh(C.Structure):
    """b2s_mesh (include/b200solve.h): peer-memory communication of a shard."""
    _fields_ = [("rank", _I), ("nranks", _I), ("nghost", _I), ("ghost_owner", _P),
                ("ghost_row", _P), ("nnbr", _I), ("nbr", _P), ("peer_x", _P),
                ("peer_phat", _P), ("peer_shat", _P), ("flags", _P), ("peer_flags", _P),
                ("mbox", _P), ("peer_mbox", _P), ("seq_base", C.c_longlong),
                ("shared_device", _I), ("host_barrier", _P), ("host_barrier_ctx", _P),
                ("nbnd", _I), ("bnd_row", _P), ("bnd_ptr", _P), ("bnd_col", _P), ("bnd_val", _P),
                ("full_sp", _P), ("full_cols", _P), ("full_vals", _P),
                ("timeout_ns", C.c_longlong)]


BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)   # 0 = ok; nonzero: this host thread failed


class BicgResult(C.Structure):
    _fields_ = [("converged", _I), ("reason", _I), ("graph_launches", _I),
                ("kernels_per_iteration", _I), ("iterations", C.c_double),
                ("initial_norm", C.c_double), ("final_norm", C.c_double)]


# name -> (restype, argtypes); mirrors include/b200solve.h
SIGNATURES = {
    "b2s_find_diagonal": (_I, [_I, _P, _P, _P, _PI, _P]),
    "b2s_level_schedule": (_I, [_I, _P, _P, _P, _PI, _P]),
    "b2s_graph_color": (_I, [_I, _P, _P, _P, _PI, _P]),
    "b2s_level_schedule_hint": (_I, [_I, _P, _P, _I, _I, _P, _P, _P, _P]),
    "b2s_graph_color_hint": (_I, [_I, _P, _P, _I, _I, _P, _P, _P, _P]),
    "b2s_analysis_trace": (_I, [_I, _I, _P, _P, _P, _P, _P]),
    "b2s_plan_from_groups": (_I, [_I, _P, _I, _P, _P, _P, _P]),
    "b2s_permute_bsr": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "b2s_gather_rows": (_I, [_I, _I, _P, _P, _P, _P]),
    "b2s_narrow_index": (_I, [_LL, _P, _P, C.POINTER(C.c_int), _P]),
    "b2s_gather_blocks": (_I, [_LL, _I, _P, _P, _P, _P]),
    "b2s_slices_plain": (_I, [_I, _P, _P, _P]),
    "b2s_slices_grouped_count": (_I, [_I, _P, _P, _PI, _P]),
    "b2s_slices_grouped_fill": (_I, [_I, _I, _P, _P, _P, _P, _P]),
    "b2s_sell_offsets": (_I, [_I, _P, _P, _P, _P, _I, _P, _PLL, _P]),
    "b2s_sell_offsets_ex": (_I, [_I, _P, _P, _P, _P, _I, _P, C.POINTER(C.c_longlong),
                                 C.POINTER(C.c_int), _P]),
    "b2s_sell_fill": (_I, [_I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _P]),
    "b2s_diag_tiles": (_I, [_I, _I, _P, _P, _P, _P, _P]),
    "b2s_sell_fill_src": (_I, [_I, _I, _P, _P, _P, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P]),
    "b2s_factor_2colour": (_I, [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                _PI, _P]),
    "b2s_factor_2colour_async": (_I, [_I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                      _P, _P, _P, _P]),
    "b2s_factor_2colour_combined": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                         _P]),
    "b2s_slice_conflicts": (_I, [_I, _P, _P, _P, _P, _PI, _P]),
    "b2s_spmv": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "b2s_ilu0_factor": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _PI, _P]),
    "b2s_ilu0_symbolic": (_I, [_I, _I, _P, _P, _P, C.POINTER(C.c_void_p), _P]),
    "b2s_ilu0_numeric": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _PI, _P]),
    "b2s_ilu0_symbolic_free": (_I, [_P, _P]),
    "b2s_ilu0_apply": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                            _I, _I, _P, _P]),
    "b2s_fill_sentinel": (_I, [_LL, _P, _P]),
    "b2s_dot_chunked": (_I, [_LL, _P, _P, _P, _P, _P]),
    "b2s_partition_greedy": (_I, [_LL, _LL, _P, _P, _P, _LL, _P]),
    "b2s_gw_workspace_bytes": (_LL, [_I, _I, _I, _I, _I, _I, _I]),
    "b2s_gw_create": (_I, [_I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _LL,
                           C.POINTER(C.c_void_p), _P]),
    "b2s_gw_fill": (_I, [_P, _P, _P, _P]),
    "b2s_gw_destroy": (_I, [_P]),
    "b2s_gw_factor_workspace_bytes": (_LL, [_P]),
    "b2s_gw_factor": (_I, [_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _LL, _P]),
    "b2s_gw_unpack_lu": (_I, [_P, _P, _P, _P, _P]),
    "b2s_gw_apply": (_I, [_I, _P, _P, _P, _P]),
    "b2s_gw_trace": (_I, [_P, _P, _LL, C.POINTER(C.c_longlong), _P]),
    "b2s_wells_apply": (_I, [_P, _P, _P, _P, _P]),
    "b2s_fuse_check": (_I, [_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _PI, _P]),
    "b2s_ilu0_apply_phased": (_I, [_I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P,
                                   _P, _P, _P, _P]),
    "b2s_tiles_trace": (_I, [_P, _P, _I]),
    "b2s_tiles_create": (_I, [_I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I,
                              C.POINTER(C.c_void_p), _P]),
    "b2s_tiles_destroy": (_I, [_P]),
    "b2s_tiles_apply": (_I, [_I, _P, _P, _P, _P, _I, _P]),
    "b2s_dot": (_I, [_LL, _P, _P, _I, _P, _P, _P]),
    "b2s_mesh_mbox_bytes": (_LL, [_I]),
    "b2s_bicgstab_workspace_layout": (_I, [_I, _I, _I, _PLL, _PLL]),
    "b2s_bicgstab_workspace_bytes_mesh": (_LL, [_I, _I, _I, _I]),
    "b2s_ipc_handle": (_I, [_P, _P, _PLL]),
    "b2s_ipc_open": (_I, [_P, _LL, C.POINTER(C.c_void_p)]),
    "b2s_ipc_close": (_I, [_P]),
    "b2s_all_finite": (_I, [_LL, _P, _P, _P]),
    "b2s_reduce": (_I, [_P, _I, _P, _P]),
    "b2s_vec_p": (_I, [_LL, _I, C.c_double, C.c_double, _P, _P, _P, _P, _P]),
    "b2s_vec_s": (_I, [_LL, C.c_double, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "b2s_vec_r": (_I, [_LL, C.c_double, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "b2s_bicgstab_workspace_bytes": (_LL, [_I, _I, _I]),
    "b2s_bicgstab": (_I, [C.POINTER(BicgArgs), C.POINTER(BicgResult)]),
    "b2s_jacobi_pattern": (_I, [_I, _P, _P, _P, _P, _PI, _P]),
    "b2s_jacobi_fill": (_I, [_I, _P, _P, _P, _P, _P, _P, _P]),
    "b2s_version": (C.c_char_p, []),
    "b2s_retain_pool_memory": (_I, [_I]),
}

_lock = threading.Lock()
_lib = None


def load(path: Path | str | None = None):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_2309_11488_b200.build` "
                "(this package has no CPU fallback)")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


class PeerTimeout(RuntimeError):
    """A sharded solve's peer did not post within the mesh timeout (dead,
    hung or misconfigured peer), or some rank aborted: B2S_PEER_TIMEOUT."""


def check(rc: int, what: str, row: int | None = None):
    """Map a C status onto the reference's exceptions (bs/errors.py)."""
    if rc == OK:
        return
    if rc == SHAPE:
        raise ShapeError(f"{what}: inconsistent sizes")
    if rc == MISSING_DIAGONAL:
        raise MissingDiagonal(int(row if row is not None else -1))
    if rc == SINGULAR_PIVOT:
        raise SingularPivot(int(row if row is not None else -1))
    if rc == UNSUPPORTED:
        raise ShapeError(f"{what}: block size outside 1..4 is not supported on the device")
    if rc == PEER_TIMEOUT:
        raise PeerTimeout(f"{what}: a peer shard did not answer in time (or aborted); "
                          "the mesh left its loop on every rank")
    raise RuntimeError(f"{what}: CUDA error (status {rc})")
