"""Stage the reference's own test suite for the drop-in conformance run.

Copies /root/reference/pkg/tests/*.py (all but test_cli.py: the CLI is out
of scope) into tests/ref_suite/_staged/, which is git-ignored (no reference
source enters the repo's history) but not gpurun-ignored, so the files travel
to the GPU box with the snapshot.  Called by __graft_entry__.build() when
/root/reference exists; the files are copied byte for byte -- the point of
the run is that the reference's tests are unmodified.  Test infrastructure.
"""

from __future__ import annotations

import hashlib
import json
import shutil
from pathlib import Path

REF_TESTS = Path("/root/reference/pkg/tests")
HERE = Path(__file__).resolve().parent
STAGED = HERE / "_staged"
EXCLUDE = {"test_cli.py"}


def stage(src: Path = REF_TESTS, dst: Path = STAGED) -> bool:
    if not src.is_dir():
        return False
    dst.mkdir(exist_ok=True)
    manifest = {}
    for f in sorted(src.glob("*.py")):
        if f.name in EXCLUDE:
            continue
        shutil.copyfile(f, dst / f.name)
        manifest[f.name] = hashlib.sha256(f.read_bytes()).hexdigest()[:16]
    (dst / "MANIFEST.json").write_text(json.dumps(
        {"source": str(src), "excluded": sorted(EXCLUDE), "sha256_16": manifest},
        indent=1) + "\n")
    return True


if __name__ == "__main__":
    print("staged" if stage() else f"{REF_TESTS} missing: nothing staged")
