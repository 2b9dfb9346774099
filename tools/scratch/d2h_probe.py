import time, torch, json
torch.cuda.init()
v = torch.rand(3_000_000, dtype=torch.float64, device="cuda")
res = {}
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts=[]
    for _ in range(reps):
        t0=time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append((time.perf_counter()-t0)*1e3)
    return round(min(ts),3), round(sorted(ts)[len(ts)//2],3)
keep=[]
def alloc_keep():
    o=torch.empty(3_000_000, dtype=torch.float64, pin_memory=True); o.copy_(v, non_blocking=True); torch.cuda.current_stream().synchronize(); keep.append(o.numpy())
def alloc_free():
    o=torch.empty(3_000_000, dtype=torch.float64, pin_memory=True); o.copy_(v, non_blocking=True); torch.cuda.current_stream().synchronize(); return o.numpy()
buf=torch.empty(3_000_000, dtype=torch.float64, pin_memory=True)
def reuse():
    buf.copy_(v, non_blocking=True); torch.cuda.current_stream().synchronize()
def alloc_only():
    keep.append(torch.empty(3_000_000, dtype=torch.float64, pin_memory=True))
res["alloc_keep"]=t(alloc_keep); res["alloc_free"]=t(alloc_free); res["reuse"]=t(reuse); res["alloc_only"]=t(alloc_only)
print(json.dumps(res))
