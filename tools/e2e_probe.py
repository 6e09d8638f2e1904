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
