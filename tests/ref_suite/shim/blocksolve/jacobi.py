"""`blocksolve.jacobi` shim -> paper_2309_11488_b200.jacobi (test infrastructure)."""
from paper_2309_11488_b200.jacobi import *  # noqa: F401,F403
from paper_2309_11488_b200 import jacobi as _impl

def __getattr__(name):
    return getattr(_impl, name)
