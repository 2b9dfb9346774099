"""The C-ABI library loads and exports every symbol include/b200solve.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import re
from pathlib import Path

from paper_2309_11488_b200 import _lib
from paper_2309_11488_b200.build import build_library

HEADER = Path(__file__).resolve().parents[1] / "include" / "b200solve.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(b2s_\w+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    path = build_library()
    lib = ctypes.CDLL(str(path))
    names = declared()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared()) == set(_lib.SIGNATURES)


def test_version_and_arch():
    lib = _lib.load()
    assert b"sm_100a" in lib.b2s_version()


def test_cubin_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
