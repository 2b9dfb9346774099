"""Phase tracing for the solve pipeline (the reference only
times with perf_counter).

Every phase opens an NVTX range (visible in Nsight / ncu --nvtx).  With
``B2S_TRACE=1`` (or ``enable()``) phases also record host wall time and a
CUDA event pair on the current stream -- no extra synchronisation -- and
``solve_with_fallback`` attaches ``report.phases = {name: (host_ms, gpu_ms)}``.
"""

from __future__ import annotations

import os
import time
from contextlib import contextmanager

import torch

_enabled = os.environ.get("B2S_TRACE", "0") == "1"
_records: list | None = None


def enable(on: bool = True):
    global _enabled
    _enabled = on


def enabled() -> bool:
    return _enabled


def start():
    """Begin collecting phases for one solve."""
    global _records
    _records = [] if _enabled else None


@contextmanager
def phase(name: str):
    nvtx = torch.cuda.is_available()
    if nvtx:
        torch.cuda.nvtx.range_push(name)
    rec = None
    if _records is not None:
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record()
        rec = [name, time.perf_counter(), e0, None, None]
    try:
        yield
    finally:
        if rec is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            rec[3], rec[4] = time.perf_counter(), e1
            _records.append(rec)
        if nvtx:
            torch.cuda.nvtx.range_pop()


def finish() -> dict | None:
    """{phase: (host_ms, gpu_ms)} of the phases since start() (synchronises)."""
    global _records
    if _records is None:
        return None
    torch.cuda.synchronize()
    out = {}
    for name, h0, e0, h1, e1 in _records:
        out[name] = (round((h1 - h0) * 1e3, 3), round(e0.elapsed_time(e1), 3))
    _records = None
    return out
