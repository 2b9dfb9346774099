"""`blocksolve.io` shim: the reference's bs/io.py is split here into the
synthetic generator (paper_2309_11488_b200.synthetic) and the Matrix Market
reader/writer (paper_2309_11488_b200.mmio).  Test infrastructure."""
from paper_2309_11488_b200.synthetic import GeneratorSpec, SystemBundle, generate  # noqa: F401
from paper_2309_11488_b200.mmio import (BundleMeta, read_system, rhs_path,  # noqa: F401
                                        wells_path, write_system)
