"""Test infrastructure: the CPU oracle for the ILU0-BiCGStab path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package -- as the checker or the
timed CPU baseline, never as part of the product.  See port.py.
"""
