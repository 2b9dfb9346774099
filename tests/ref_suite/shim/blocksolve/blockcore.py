"""`blocksolve.blockcore` shim -> paper_2309_11488_b200.blockcore (test infrastructure)."""
from paper_2309_11488_b200.blockcore import *  # noqa: F401,F403
from paper_2309_11488_b200 import blockcore as _impl

def __getattr__(name):
    return getattr(_impl, name)
