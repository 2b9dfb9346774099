import sys, time, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200.distributed import local_solver
from paper_2309_11488_b200 import bridge as B, ilu0 as I, _device as D
shards, comm = local_solver(P.GeneratorSpec(100, 100, 100, seed=0), 1, P.Backend.GRAPH_COLORED)
s = shards[0]
def tick(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize(); return out, round((time.perf_counter()-t0)*1e3, 3)
for rep in range(3):
    plan, t_plan = tick(lambda: B.plan_device(P.Backend.GRAPH_COLORED, s.pbsr.pat))
    fact, t_fact = tick(lambda: I.factor_device(s.pmat, plan, s.pbsr))
    _, t_setup = tick(lambda: s.setup(P.Backend.GRAPH_COLORED))
print(json.dumps({"plan": t_plan, "factor": t_fact, "shard_setup_total": t_setup}))
