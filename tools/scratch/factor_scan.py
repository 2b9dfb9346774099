"""Level factorisation on C4: scan CTAs per SM x warps per CTA (env knobs of
launch_numeric); prints the numeric kernel's CUDA-event time per config."""
import json, os, subprocess, sys
sys.path.insert(0, '/root/repo')
code = r'''
import sys, json, torch
sys.path.insert(0, "/root/repo")
import paper_2309_11488_b200 as P
from paper_2309_11488_b200 import _device as D
from paper_2309_11488_b200.bridge import plan_device
from paper_2309_11488_b200.ilu0 import factor_device
a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
plan = plan_device(P.Backend.LEVEL_SCHEDULED, bsr.pat)
st = torch.cuda.current_stream()
for _ in range(2): factor_device(a, plan, bsr)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(5): factor_device(a, plan, bsr)
e1.record(st); torch.cuda.synchronize()
print(json.dumps(e0.elapsed_time(e1) / 5))
'''
res = {}
for ctas in (1, 2, 3):
    for warps in (2, 3, 4, 6, 8):
        env = dict(os.environ, B2S_FACTOR_CTAS_PER_SM=str(ctas), B2S_FACTOR_WARPS=str(warps))
        out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        try:
            res[f"c{ctas}_w{warps}"] = round(float(out.stdout.strip().splitlines()[-1]), 3)
        except Exception:
            res[f"c{ctas}_w{warps}"] = out.stderr[-200:]
out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
res["default"] = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-200:]
print(json.dumps(res))
