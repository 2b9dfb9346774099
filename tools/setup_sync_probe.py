"""Host synchronisations inside one C4 setup (plan + factorisation + operator
layouts): every CUDA runtime call that waits for the device, with its host
duration and the Python frames that issued it (torch profiler, CPU + CUDA).

python tools/setup_sync_probe.py [color|level]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import paper_2309_11488_b200 as P  # noqa: E402
from paper_2309_11488_b200 import _device as D  # noqa: E402
from paper_2309_11488_b200.bridge import DeviceSolver  # noqa: E402

backend = sys.argv[1] if len(sys.argv) > 1 else "color"
a = P.generate(P.GeneratorSpec(100, 100, 100, seed=0)).a
bsr = D.DevBSR.upload(a)
cfg = P.SolverConfig(backend=P.Backend.from_name(backend))
solver = None
for _ in range(3):
    bsr.pat.__dict__.pop("_diag", None)
    solver = None
    solver = DeviceSolver(a, bsr, cfg).setup()
torch.cuda.synchronize()
bsr.pat.__dict__.pop("_diag", None)
solver = None
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts, with_stack=True) as prof:
    solver = DeviceSolver(a, bsr, cfg).setup()
    torch.cuda.synchronize()
# every b2s_* call and torch host read: host duration + the calling frame
import time  # noqa: E402
import traceback  # noqa: E402

calls = []
L = D.lib()
for name in dir(L):
    if not name.startswith("b2s_"):
        continue
    fn = getattr(L, name)

    def wrap(*args, _fn=fn, _name=name):
        t = time.perf_counter()
        r = _fn(*args)
        calls.append((_name, (time.perf_counter() - t) * 1e6, _caller()))
        return r
    setattr(L, name, wrap)


def _caller():
    for fr in reversed(traceback.extract_stack()[:-2]):
        if "paper_2309" in fr.filename:
            return f"{fr.filename.split('/')[-1]}:{fr.lineno}:{fr.name}"
    return "?"


for meth in ("item", "cpu", "tolist"):
    orig = getattr(torch.Tensor, meth)

    def wrapm(self, *args, _o=orig, _m=meth, **kw):
        t = time.perf_counter()
        r = _o(self, *args, **kw)
        calls.append((f"Tensor.{_m}", (time.perf_counter() - t) * 1e6, _caller()))
        return r
    setattr(torch.Tensor, meth, wrapm)
bsr.pat.__dict__.pop("_diag", None)
solver = None
torch.cuda.synchronize()
t_all = time.perf_counter()
solver = DeviceSolver(a, bsr, cfg).setup()
torch.cuda.synchronize()
print(json.dumps({"setup_wall_ms": round((time.perf_counter() - t_all) * 1e3, 3)}))
for name, us, where in calls:
    print(json.dumps({"call": name, "host_us": round(us, 1), "at": where}))
waits = ("cudaStreamSynchronize", "cudaMemcpy", "cudaMemcpyAsync", "cudaDeviceSynchronize",
         "cudaEventSynchronize", "aten::item", "aten::_local_scalar_dense", "aten::to",
         "aten::copy_")
rows = []
for ev in prof.events():
    if ev.name in waits or "Synchronize" in ev.name:
        stack = [f for f in (ev.stack or []) if "paper_2309" in f][:4]
        rows.append({"name": ev.name, "host_us": round(ev.cpu_time_total, 1),
                     "t_us": round(ev.time_range.start, 1), "stack": stack})
rows.sort(key=lambda r: r["t_us"])
t0 = rows[0]["t_us"] if rows else 0
for r in rows:
    r["t_us"] = round(r["t_us"] - t0, 1)
    print(json.dumps(r))
gpu = sum(e.device_time_total for e in prof.key_averages() if e.device_time_total) / 1e3
print(json.dumps({"gpu_kernel_ms_total": round(gpu, 3)}))
# device timeline: idle gaps between consecutive GPU activities (what the
# host synchronisations cost), with the activity that ended each gap
dev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
             key=lambda e: e.time_range.start)
if dev:
    t0, last_end = dev[0].time_range.start, dev[0].time_range.end
    idle = 0.0
    for e in dev[1:]:
        gap = e.time_range.start - last_end
        if gap > 5:
            idle += gap
            print(json.dumps({"gap_us": round(gap, 1), "at_us": round(e.time_range.start - t0, 1),
                              "next": e.name[:60]}))
        last_end = max(last_end, e.time_range.end)
    print(json.dumps({"span_us": round(last_end - t0, 1), "idle_us": round(idle, 1)}))
