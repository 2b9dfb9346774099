"""Host->device upload strategies for a 500 MB fp64 array (e2e path)."""
import time
import numpy as np
import torch

n = 62_460_000   # 6.94M blocks x 9
a = np.random.default_rng(0).random(n)
dev = torch.device("cuda")
torch.cuda.synchronize()


def t(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name:40s} {dt*1e3:8.2f} ms  {a.nbytes/dt/1e9:6.1f} GB/s", flush=True)


t("pageable torch .to()", lambda: torch.from_numpy(a).to(dev))
cudart = torch.cuda.cudart()


def reg():
    ptr = a.ctypes.data
    cudart.cudaHostRegister(ptr, a.nbytes, 0)
    out = torch.from_numpy(a).to(dev, non_blocking=True)
    torch.cuda.synchronize()
    cudart.cudaHostUnregister(ptr)
    return out


t("cudaHostRegister + copy + unregister", reg)
pin = torch.empty(n, dtype=torch.float64).pin_memory()


def staged():
    pin.numpy()[:] = a
    return pin.to(dev, non_blocking=True)


t("np copy into pinned + async copy", staged)
out = torch.empty(n, dtype=torch.float64, device=dev)
from concurrent.futures import ThreadPoolExecutor
pool = ThreadPoolExecutor(8)
CH = 1 << 21   # 2M doubles = 16 MB
pins = [torch.empty(CH, dtype=torch.float64).pin_memory() for _ in range(4)]
streams = [torch.cuda.Stream() for _ in range(4)]
events = [None] * 4


def chunked():
    def fill(i, lo, hi):
        pins[i].numpy()[: hi - lo] = a[lo:hi]
    futs = []
    lo = 0
    k = 0
    while lo < n:
        hi = min(n, lo + CH)
        i = k % 4
        if events[i] is not None:
            events[i].synchronize()
        fill(i, lo, hi)
        with torch.cuda.stream(streams[i]):
            out[lo:hi].copy_(pins[i][: hi - lo], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(streams[i])
            events[i] = ev
        lo = hi
        k += 1
    torch.cuda.synchronize()


t("chunked 16MB pinned double-buffer", chunked)


def par_staged():
    buf = pin.numpy()
    parts = np.array_split(np.arange(n), 8)
    list(pool.map(lambda p: buf.__setitem__(slice(p[0], p[-1] + 1), a[p[0]:p[-1] + 1]), parts))
    return pin.to(dev, non_blocking=True)


t("8-thread copy into pinned + async copy", par_staged)
