"""`blocksolve.analysis` shim -> paper_2309_11488_b200.analysis (test infrastructure)."""
from paper_2309_11488_b200.analysis import *  # noqa: F401,F403
from paper_2309_11488_b200 import analysis as _impl

def __getattr__(name):
    return getattr(_impl, name)
