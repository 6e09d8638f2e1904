"""Development aid: host->device paths for a numpy float64 vector (the
reference calling convention) and device->host back into numpy."""
import time, sys
import numpy as np, torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3060300
a = np.random.default_rng(0).standard_normal(n)
dev = torch.device("cuda")
d = torch.empty(n, dtype=torch.float64, device=dev)
print("torch threads", torch.get_num_threads())
def T(name, fn, reps=20):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); s = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append(time.perf_counter() - s)
    print(f"{name:34s} median {np.median(ts)*1e3:7.3f} ms  min {min(ts)*1e3:7.3f}", flush=True)
T("pageable to(dev)", lambda: d.copy_(torch.from_numpy(a)))
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
T("pinned DMA only", lambda: d.copy_(pin, non_blocking=True))
T("memcpy np->pinned (torch copy_)", lambda: pin.copy_(torch.from_numpy(a)))
T("np.copyto np->pinned", lambda: np.copyto(pin.numpy(), a))
def staged(k):
    src = torch.from_numpy(a)
    def f():
        step = (n + k - 1) // k
        for i in range(0, n, step):
            pin[i:i + step].copy_(src[i:i + step])
            d[i:i + step].copy_(pin[i:i + step], non_blocking=True)
    return f
for k in (4, 8, 16, 32):
    T(f"staged chunks={k}", staged(k))
cud = torch.cuda.cudart()
def reg():
    p = a.ctypes.data
    cud.cudaHostRegister(p, a.nbytes, 0)
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    cud.cudaHostUnregister(p)
T("cudaHostRegister+DMA+unregister", reg)
# D2H
T("d2h pageable .cpu().numpy()", lambda: d.cpu().numpy())
T("d2h pinned copy (caching alloc)", lambda: torch.empty(n, dtype=torch.float64, pin_memory=True).copy_(d).numpy())
out = np.empty(n)
def d2h_staged(k):
    def f():
        step = (n + k - 1) // k
        evs = []
        for i in range(0, n, step):
            pin[i:i + step].copy_(d[i:i + step], non_blocking=True)
            e = torch.cuda.Event(); e.record(); evs.append((i, e))
        for i, e in evs:
            e.synchronize()
            np.copyto(out[i:i + step], pin.numpy()[i:i + step])
    return f
for k in (4, 8, 16):
    T(f"d2h staged chunks={k} into np", d2h_staged(k))
