"""Build libb200solve.so (sm_100a) in-tree with nvcc.

The shared library is the product's only compute path; it is compiled for
``sm_100a`` exclusively (``-gencode arch=compute_100a,code=sm_100a``) and
loaded through ctypes by ``_lib.py``.  Built artefacts live next to the
sources (git-ignored, but shipped to the GPU box by gpurun).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIB = PKG / "libb200solve.so"
SOURCES = ["analysis.cu", "spmv.cu", "factor.cu", "ilu0.cu", "fused.cu", "factor2c.cu", "tiles.cu", "krylov.cu",
           "jacobi.cu", "wells.cu", "refdot.cu", "gridwave.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


OBJ = ROOT / "build" / "obj"


def _newer(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _headers():
    return list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))


def _stale() -> bool:
    return _newer(LIB, [CSRC / s for s in SOURCES] + _headers())


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Compile each source to an object in parallel (only the stale ones),
    then link the shared library."""
    if not force and not _stale():
        return LIB
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr = _headers()
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    compile_flags += os.environ.get("B2S_EXTRA_NVCC", "").split()   # e.g. -DB2S_GW_TRACE_BUILD
    procs = []
    for src in SOURCES:
        obj = OBJ / (Path(src).stem + ".o")
        if force or _newer(obj, [CSRC / src] + hdr):
            cmd = [nvcc(), *compile_flags, f"-I{INCLUDE}", f"-I{CSRC}", "-c", str(CSRC / src),
                   "-o", str(obj) + ".tmp"]
            procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                     stderr=subprocess.PIPE, text=True)))
    logs, failed = [], []
    for src, obj, p in procs:
        out, err = p.communicate()
        logs.append(f"== {src}\n{out}{err}")
        if p.returncode != 0:
            failed.append((src, err))
        else:
            os.replace(str(obj) + ".tmp", obj)
    log = CSRC / "ptxas.log"
    log.write_text("\n".join(logs))
    if failed:
        for src, err in failed:
            sys.stderr.write(f"== {src}\n{err[-6000:]}")
        raise RuntimeError(f"nvcc failed on {[f[0] for f in failed]}; see {log}")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
           *[str(OBJ / (Path(s).stem + ".o")) for s in SOURCES], "-o", str(LIB) + ".tmp"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-6000:])
        raise RuntimeError(f"link failed ({proc.returncode})")
    os.replace(str(LIB) + ".tmp", LIB)
    if verbose:
        sys.stderr.write("\n".join(logs))
    return LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
