"""`blocksolve.krylov` shim -> paper_2309_11488_b200.krylov (test infrastructure)."""
from paper_2309_11488_b200.krylov import *  # noqa: F401,F403
from paper_2309_11488_b200 import krylov as _impl

def __getattr__(name):
    return getattr(_impl, name)
