import sys, time, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D, synthetic as S
from paper_2309_11488_b200.bridge import plan_device, DeviceSolver
from paper_2309_11488_b200.ilu0 import factor_device
from paper_2309_11488_b200.krylov import DeviceKrylov
def tick(fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); out = fn(); torch.cuda.synchronize()
    return out, round((time.perf_counter() - t0) * 1e3, 3)
order = sys.argv[1:] or ["c3", "c4"]
for name in order:
    bnd = S.generate_heterogeneous(92, 224, 17, sigma_k=1.0, diagonal_boost=1e-2) if name == "c3" else \
        P.generate(P.GeneratorSpec(100, 100, 100, seed=0))
    a = bnd.a
    bsr = D.DevBSR.upload(a)
    for rep in range(3):
        plan, t1 = tick(lambda: plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat))
        f, t2 = tick(lambda: factor_device(a, plan, bsr))
        kr, t3 = tick(lambda: DeviceKrylov.build(a, f))
        s, t4 = tick(lambda: DeviceSolver(a, bsr, P.SolverConfig(backend=P.Backend.LEVEL_SCHEDULED)).setup())
        print(json.dumps({"cfg": name, "rep": rep, "plan": t1, "factor": t2, "krylov_build": t3,
                          "solver_setup": t4, "hint": getattr(bsr.pat, "hint_used", None)}), flush=True)
