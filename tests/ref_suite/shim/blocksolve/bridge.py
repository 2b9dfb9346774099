"""`blocksolve.bridge` shim -> paper_2309_11488_b200.bridge (test infrastructure)."""
from paper_2309_11488_b200.bridge import *  # noqa: F401,F403
from paper_2309_11488_b200 import bridge as _impl

def __getattr__(name):
    return getattr(_impl, name)
