"""`blocksolve.wells` shim -> paper_2309_11488_b200.wells (test infrastructure)."""
from paper_2309_11488_b200.wells import *  # noqa: F401,F403
from paper_2309_11488_b200 import wells as _impl

def __getattr__(name):
    return getattr(_impl, name)
