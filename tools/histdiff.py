"""Development aid: residual-history drift of the device solver vs the oracle,
next to the drift of an oracle variant with a re-ordered FP32 fine apply
(FP64 accumulation, rounded once) -- the legitimate-noise band."""
import sys, warnings
import numpy as np
sys.path.insert(0, ".")
import paper_2604_26441_b200 as P
from oracle import simp_oracle as O

dims = tuple(int(v) for v in sys.argv[1].split("x")) if len(sys.argv) > 1 else (16, 8, 8)
kind = sys.argv[2] if len(sys.argv) > 2 else "binary"
p = float(sys.argv[3]) if len(sys.argv) > 3 else 3.0
vf = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
g = P.build_cantilever(*dims)
op = P.FineOperator(g, P.simp_modulus(P.make_state(kind, *dims, vf=vf, seed=42), p))
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    h = P.build_hierarchy(op, 4, "fp32")
b = g.load[g.free_dofs]
rep = P.pcg(op.matvec, h.vcycle, b, P.SolverConfig(tol=1e-6, maxiter=200))
og, E, ke = O.problem(*dims, kind=kind, vf=vf, p=p, seed=42)
ref, oh = O.solve(og, E, ke, "fp32")
# perturbed oracle: FP32 apply with FP64 accumulation rounded once
orig = O.fine_apply
def pert(g_, E_, ke_, u, tag="fp64"):
    if tag != "fp32":
        return orig(g_, E_, ke_, u, tag)
    return orig(g_, E_, ke_, np.asarray(u, np.float64), "fp64").astype(np.float32)
O.fine_apply = pert
alt, _ = O.solve(og, E, ke, "fp32")
O.fine_apply = orig
k = min(len(rep.residual_history), len(ref.residual_history), len(alt.residual_history))
d_dev = np.abs(np.array(rep.residual_history[:k]) / np.array(ref.residual_history[:k]) - 1)
d_alt = np.abs(np.array(alt.residual_history[:k]) / np.array(ref.residual_history[:k]) - 1)
print(dims, kind, p, vf, "iters dev/ref/perturbed-ref:", rep.iterations, ref.iterations, alt.iterations)
for i in list(range(0, k, max(1, k // 12))) + [k - 1]:
    print(f"  it {i:3d} dev-ref {d_dev[i]:.2e}  pert-ref {d_alt[i]:.2e}")
print("  max dev-ref", d_dev.max(), "max pert-ref", d_alt.max())
