"""`blocksolve.ilu0` shim -> paper_2309_11488_b200.ilu0 (test infrastructure)."""
from paper_2309_11488_b200.ilu0 import *  # noqa: F401,F403
from paper_2309_11488_b200 import ilu0 as _impl

def __getattr__(name):
    return getattr(_impl, name)
