"""`blocksolve.errors` shim -> paper_2309_11488_b200.errors (test infrastructure)."""
from paper_2309_11488_b200.errors import *  # noqa: F401,F403
from paper_2309_11488_b200 import errors as _impl

def __getattr__(name):
    return getattr(_impl, name)
