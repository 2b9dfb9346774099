"""Level-plan sync-free sweeps on C4: scan (CTAs per SM, warps per CTA,
ticket mode, back-off) through Ilu0Factorization.sweep_flags."""
import json, sys
sys.path.insert(0, '/root/repo')
import torch
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D
from paper_2309_11488_b200.bridge import plan_device
from paper_2309_11488_b200.ilu0 import factor_device

a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
f = factor_device(a, plan, bsr)
m = a.num_block_rows * 3
x = torch.rand(m, dtype=torch.float64, device="cuda")
z = torch.empty(m, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
ref = None
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps): fn()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
out = {}
for per_sm in (1,):
    for warps in (1, 2, 3, 4, 5):
        for static in (0,):
            for nap in (0, 1):
                flags = (per_sm << 4) | (warps << 8) | static | nap
                f.sweep_flags = flags
                us = t(lambda: f.apply_device(x, z))
                if ref is None: ref = z.clone()
                ok = bool(torch.equal(z, ref))
                out[f"sm{per_sm}_w{warps}_st{static}_nap{nap}"] = (round(us, 1), ok)
best = sorted(out.items(), key=lambda kv: kv[1][0])[:8]
print(json.dumps({"default_0x10": out.get("sm1_w8_st0_nap0"), "best": best}))
