"""Drop-in conformance run: the reference's own tests (staged unmodified in
_staged/ by stage.py) import `blocksolve`, which resolves to the shim in
shim/blocksolve -> paper_2309_11488_b200.  Every staged test is a GPU test
(the package has no CPU path).  Known, reasoned deviations are listed in
EXPECTED_DEVIATIONS and turned into xfail(strict=True) so a fix shows up.
"""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent
SHIM = HERE / "shim"
if str(SHIM) not in sys.path:
    sys.path.insert(0, str(SHIM))

STAGED = HERE / "_staged"

# nodeid suffix -> reason
EXPECTED_DEVIATIONS: dict[str, str] = {}


def pytest_ignore_collect(collection_path, config):
    # stage.py was not run (no /root/reference where build() ran): nothing to run
    p = Path(collection_path)
    if p.name == "shim" and p.parent == HERE:
        return True
    return None


def pytest_collection_modifyitems(config, items):
    for item in items:
        path = Path(str(item.fspath)).resolve()
        if STAGED not in path.parents:
            continue
        item.add_marker(pytest.mark.gpu)
        item.add_marker(pytest.mark.ref_suite)
        for suffix, why in EXPECTED_DEVIATIONS.items():
            if item.nodeid.endswith(suffix):
                item.add_marker(pytest.mark.xfail(reason=why, strict=True))
