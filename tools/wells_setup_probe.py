import sys, time, cProfile, pstats
sys.path.insert(0,'/root/repo')
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D
from paper_2309_11488_b200.bridge import DeviceSolver
g = P.generate(P.GeneratorSpec(100,100,100, seed=0, well_count=20, well_depth=10))
a = g.a
bsr = D.DevBSR.upload(a)
cfg = P.SolverConfig(backend=P.Backend.GRAPH_COLORED)
for w in (None, g.wells):
    for _ in range(3):
        s = None; torch.cuda.synchronize(); t0=time.perf_counter()
        s = DeviceSolver(a, bsr, cfg, wells=w).setup(); torch.cuda.synchronize()
        t = time.perf_counter()-t0
    print('wells' if w else 'plain', round(t*1e3,2), 'ms')
pr = cProfile.Profile(); pr.enable()
s = None; s = DeviceSolver(a, bsr, cfg, wells=g.wells).setup(); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats('cumulative').print_stats(18)
