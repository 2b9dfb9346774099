"""Host-side profile of DeviceSolver.setup (colour, C4): where the non-kernel
time of the setup goes."""
import cProfile, pstats, sys, time
sys.path.insert(0, '/root/repo')
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D
from paper_2309_11488_b200.bridge import DeviceSolver
g = P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
bsr = D.DevBSR.upload(g.a)
cfg = P.SolverConfig(backend=P.Backend.GRAPH_COLORED)
for _ in range(3):
    DeviceSolver(g.a, bsr, cfg).setup()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    DeviceSolver(g.a, bsr, cfg).setup()
torch.cuda.synchronize()
print("setup ms", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    DeviceSolver(g.a, bsr, cfg).setup()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
