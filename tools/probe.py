"""Quick timing probe (development aid): fine applies and one full solve."""
import sys, time, warnings
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from paper_2604_26441_b200 import _dev, _native

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
g = P.build_cantilever(N, N, N)
t0 = time.perf_counter()
op = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", N, N, N, vf=0.5), 3.0))
torch.cuda.synchronize(); print(f"op create {time.perf_counter()-t0:.3f}s")
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
for tag, dt in ((P.PrecisionTag.FP32, np.float32), (P.PrecisionTag.FP64, np.float64)):
    u, _ = _dev.as_device(np.random.default_rng(0).standard_normal(g.n_free), dt)
    y = _dev.empty(g.n_free, dt)
    times = []
    for it in range(8):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _native.check(op._lib.sg_fine_apply(op._h, tag.code, _dev.ptr(u), _dev.ptr(y), _dev.stream()))
        e.record(); torch.cuda.synchronize(); times.append(s.elapsed_time(e))
    print(f"fine apply {tag.value} (free layout incl. scatter/gather): {np.median(times[3:])*1e3:.1f} us")
t0 = time.perf_counter()
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
torch.cuda.synchronize(); print(f"setup {time.perf_counter()-t0:.3f}s levels {[l.n_free for l in h.levels]} mode {h.coarsest.mode} lams {[round(l.lam_max,4) for l in h.levels]}")
b = g.load[g.free_dofs]
for trial in range(3):
    rep = P.pcg(op.matvec, h.vcycle, b, P.SolverConfig(tol=1e-6, maxiter=200))
    print(f"solve {rep.wall_time:.4f}s iters {rep.iterations} true {rep.final_true_residual:.3e} conv {rep.converged}")
print("hist", [f"{v:.4e}" for v in rep.residual_history])
