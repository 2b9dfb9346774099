import json, os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D
from paper_2309_11488_b200.bridge import plan_device
from paper_2309_11488_b200.ilu0 import factor_device
a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
ref = None
for cfg in [("0", "8"), ("100", "8"), ("400", "8"), ("0", "4"), ("100", "4"), ("0", "2"), ("200", "2")]:
    os.environ["B2S_FACTOR_SLEEP"], os.environ["B2S_FACTOR_WARPS"] = cfg
    ts = []
    for _ in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        f = factor_device(a, plan, bsr)
        torch.cuda.synchronize(); ts.append((time.perf_counter() - t) * 1e3)
    same = None
    if ref is None:
        ref = f.inverted_diagonals.copy()
    else:
        same = bool((f.inverted_diagonals == ref).all())
    print(json.dumps({"sleep": cfg[0], "warps": cfg[1], "factor_ms": [round(x, 2) for x in ts], "same": same}), flush=True)
