"""Development aid: where the end-to-end (host buffers) solve time goes at 100^3."""
import sys, time, warnings
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev
N = 100
g = P.build_cantilever(N, N, N)
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
b_host = np.ascontiguousarray(g.load[g.free_dofs])
b_dev, _ = _dev.as_device(b_host)
cfg = P.SolverConfig(tol=1e-6, maxiter=200)
b_pin = torch.from_numpy(b_host).pin_memory()
x_pin = torch.empty_like(b_pin).pin_memory()
print("pinned:", b_pin.is_pinned(), x_pin.is_pinned())
def wall(f, n=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); s = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - s)
    return 1e3 * min(ts), 1e3 * np.median(ts)
print("h2d        ms", wall(lambda: b_pin.to("cuda")))
xd = b_dev.clone()
print("d2h        ms", wall(lambda: x_pin.copy_(xd)))
print("solve(dev) ms", wall(lambda: P.pcg(op.matvec, h.vcycle, b_dev, cfg)))
print("solve(pin) ms", wall(lambda: P.pcg(op.matvec, h.vcycle, b_pin, cfg)))
def e2e():
    r = P.pcg(op.matvec, h.vcycle, b_pin, cfg)
    x_pin.copy_(r.x)
print("e2e        ms", wall(e2e))
print("solve(np)  ms", wall(lambda: P.pcg(op.matvec, h.vcycle, b_host, cfg)))
from paper_2604_26441_b200 import _dev as D
print("as_device(np) ms", wall(lambda: D.as_device(b_host)))
print("back(host)    ms", wall(lambda: D.back(xd, True)))
ts = []
for _ in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    bd, _ = D.as_device(b_host); torch.cuda.synchronize(); t1 = time.perf_counter()
    r = P.pcg(op.matvec, h.vcycle, bd, cfg); torch.cuda.synchronize(); t2 = time.perf_counter()
    xo = D.back(r.x, True); t3 = time.perf_counter()
    r2 = P.pcg(op.matvec, h.vcycle, b_host, cfg); torch.cuda.synchronize(); t4 = time.perf_counter()
    ts.append([(t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3])
print("split h2d / solve / d2h / np-call ms", np.median(np.array(ts), axis=0))
import collections
acc = collections.defaultdict(list)
_orig_as, _orig_back = D.as_device, D.back
def as_dev_t(*a, **k):
    torch.cuda.synchronize(); t = time.perf_counter(); r = _orig_as(*a, **k); torch.cuda.synchronize()
    acc["as_device"].append(time.perf_counter() - t); return r
def back_t(*a, **k):
    t = time.perf_counter(); r = _orig_back(*a, **k); acc["back"].append(time.perf_counter() - t); return r
_orig_empty = torch.empty
def empty_t(*a, **k):
    t = time.perf_counter(); r = _orig_empty(*a, **k)
    if k.get("pin_memory"): acc["pinned_empty"].append(time.perf_counter() - t)
    return r
D.as_device, D.back, torch.empty = as_dev_t, back_t, empty_t
for _ in range(10):
    torch.cuda.synchronize(); t = time.perf_counter()
    P.pcg(op.matvec, h.vcycle, b_host, cfg); torch.cuda.synchronize()
    acc["call"].append(time.perf_counter() - t)
D.as_device, D.back, torch.empty = _orig_as, _orig_back, _orig_empty
print({k: round(float(np.median(v)) * 1e3, 3) for k, v in acc.items()})
