"""Matrix Market fixtures written by the UNMODIFIED reference (bs/io.py
write_system) for the reader round-trip tests.  Container only:
    python tests/golden/make_mm.py
"""
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from blocksolve.io import GeneratorSpec, generate, write_system  # noqa: E402

OUT = Path(__file__).resolve().parent / "mm"
OUT.mkdir(exist_ok=True)
write_system(generate(GeneratorSpec(3, 2, 2, well_count=1, well_depth=2, seed=44)),
             OUT / "std.mtx")
write_system(generate(GeneratorSpec(3, 3, 3, well_count=2, well_depth=3,
                                    well_kind="multisegment", seed=9)), OUT / "msw.mtx")
write_system(generate(GeneratorSpec(4, 3, 2, block_size=2, seed=7)), OUT / "b2.mtx")
print(sorted(p.name for p in OUT.iterdir()))
