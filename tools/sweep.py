"""27-case heterogeneous sweep (BASELINE configs 2/3): device FP32-GMG PCG (or
BF16-GMG FGMRES) per (vf, p) cell, optionally next to the CPU oracle.

    python tools/sweep.py 40 [--oracle] [--policy fp32|bf16] [--jacobi]
"""
import argparse, json, sys, time, warnings
sys.path.insert(0, ".")
import numpy as np
import paper_2604_26441_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("N", type=int)
ap.add_argument("--oracle", action="store_true")
ap.add_argument("--policy", default="fp32")
ap.add_argument("--jacobi", action="store_true")
ap.add_argument("--restart", type=int, default=32)
ap.add_argument("--maxiter", type=int, default=200)
args = ap.parse_args()
N = args.N
out = []
for vf in (0.2, 0.5, 0.8):
    for p in (1.5, 3.0, 4.5):
        g = P.build_cantilever(N, N, N)
        op = P.FineOperator(g, P.simp_modulus(P.make_state("binary", N, N, N, vf=vf, floor=1e-2, seed=42), p))
        b = g.load[g.free_dofs]
        t0 = time.perf_counter()
        if args.jacobi:
            rep = P.flat_jacobi_pcg(op, b, P.SolverConfig(tol=1e-6, maxiter=args.maxiter))
        else:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                h = P.build_hierarchy(op, 4, args.policy)
            method = "fgmres" if args.policy == "bf16" else "pcg"
            solver = P.fgmres if method == "fgmres" else P.pcg
            rep = solver(op.matvec, h.vcycle, b, P.SolverConfig(method=method, tol=1e-6,
                                                                 maxiter=args.maxiter, restart=args.restart))
        dt = time.perf_counter() - t0
        cell = {"vf": vf, "p": p, "iters": rep.iterations, "conv": rep.converged,
                "kind": rep.failure_kind, "true": rep.final_true_residual, "s": dt}
        if args.oracle:
            from oracle import simp_oracle as O
            og, E, ke = O.problem(N, N, N, kind="binary", vf=vf, p=p, seed=42)
            if args.jacobi:
                ref = O.jacobi_pcg(og, E, ke, og.load[og.free], 1e-6, args.maxiter)
            else:
                method = "fgmres" if args.policy == "bf16" else "pcg"
                ref, _ = O.solve(og, E, ke, args.policy, method=method, maxiter=args.maxiter,
                                 restart=args.restart)
            cell.update({"ref_iters": ref.iterations, "ref_conv": ref.converged,
                         "ref_true": ref.final_true_residual})
        out.append(cell)
        print(json.dumps(cell), flush=True)
print("device pass", sum(c["conv"] for c in out), "/ 9")
