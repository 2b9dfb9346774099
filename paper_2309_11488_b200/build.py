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
           "jacobi.cu", "wells.cu"]
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


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}",
           *[str(CSRC / s) for s in SOURCES], "-o", str(LIB) + ".tmp"]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = CSRC / "ptxas.log"
    log.write_text(proc.stdout + proc.stderr)
    if proc.returncode != 0:
        sys.stderr.write(proc.stderr[-6000:])
        raise RuntimeError(f"nvcc failed ({proc.returncode}); see {log}")
    os.replace(str(LIB) + ".tmp", LIB)
    if verbose:
        sys.stderr.write(proc.stderr)
    return LIB


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
