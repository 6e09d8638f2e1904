"""Golden fixtures for the BASELINE sweep configs, made by running the REAL reference.

Test infrastructure only (like ``make_golden.py``): it imports ``simpgmg`` from
/root/reference/pkg/src (read-only) in the build container and writes small JSON
fixtures under tests/golden/.  The ``-m gpu`` tests in
``tests/test_baseline_configs_gpu.py`` compare the sm_100a product with them on the
GPU box (where /root/reference does not exist).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_sweep.py fp32 40     # 9 cells
    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_sweep.py jacobi 60   # 9 cells
    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_sweep.py bf16 80 0-4 # cells 0..4
    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_sweep.py big 100     # history + samples

Cell recipes (all binary density, seed 42, floor 1e-2, tol 1e-6):
  fp32   -> bench/runner.py:66-88  run_solver(method="pcg") on build_gmg(precision="fp32")
  jacobi -> krylov.py:284-288      flat_jacobi_pcg, cap 200 (configs[1] comparator)
  bf16   -> bench/runner.py:319-343 cell: FP64 hierarchy -> Lanczos m=40 probe on
            vcycle64(K .) -> "bf16" hierarchy -> FGMRES(restart 50, cap 500)
  big    -> configs[3] (100^3 uniform rho=0.5 p=3) or configs[2] size (80^3): residual
            history, true residual, V-cycle and BF16/FP32 apply at strided sample indices.
"""

from __future__ import annotations

import json
import os
import sys
import time
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")
VFS = (0.2, 0.5, 0.8)
PS = (1.5, 3.0, 4.5)
CELLS = [(vf, p) for vf in VFS for p in PS]
N_SAMPLE = 4096


def _problem(S, N, vf, p, kind="binary"):
    g = S.build_cantilever(N, N, N)
    if kind == "binary":
        st = S.make_state("binary", N, N, N, vf=vf, floor=1e-2, seed=42)
    else:
        st = S.make_state("uniform", N, N, N, vf=vf)
    return g, S.FineOperator(g, S.simp_modulus(st, p))


def _rep(rep):
    return {"converged": bool(rep.converged), "iterations": int(rep.iterations),
            "failure_kind": rep.failure_kind,
            "final_true_residual": float(rep.final_true_residual),
            "residual_history": [float(v) for v in rep.residual_history]}


def _hier(S, op, policy):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return S.build_hierarchy(op, 4, policy)


def fp32(S, N):
    out = {}
    for vf, p in CELLS:
        t0 = time.time()
        g, op = _problem(S, N, vf, p)
        h = _hier(S, op, "fp32")
        rep = S.pcg(op.matvec, h.vcycle, g.load[g.free_dofs],
                    S.SolverConfig(tol=1e-6, maxiter=200))
        out[f"{vf}_{p}"] = _rep(rep)
        print(N, vf, p, rep.iterations, rep.converged, f"{time.time() - t0:.1f}s", flush=True)
    return out


def jacobi(S, N):
    out = {}
    for vf, p in CELLS:
        g, op = _problem(S, N, vf, p)
        rep = S.flat_jacobi_pcg(op, g.load[g.free_dofs], S.SolverConfig(tol=1e-6, maxiter=200))
        out[f"{vf}_{p}"] = _rep(rep)
        print(N, vf, p, rep.iterations, rep.final_true_residual, flush=True)
    return out


def bf16(S, N, cells):
    out = {}
    for i in cells:
        vf, p = CELLS[i]
        t0 = time.time()
        g, op = _problem(S, N, vf, p)
        h64 = _hier(S, op, "fp64")
        pr = S.lanczos_kappa_eff(lambda v: h64.vcycle(op.matvec_tagged(v, S.PrecisionTag.FP64)),
                                 op.n_free, 40, 0)
        h16 = _hier(S, op, "bf16")
        rep = S.fgmres(op.matvec, h16.vcycle, g.load[g.free_dofs],
                       S.SolverConfig(method="fgmres", tol=1e-6, maxiter=500, restart=50))
        d = _rep(rep)
        d.update(kappa_eff=float(pr.kappa_eff), eps_kappa=float(pr.eps_kappa),
                 lambda_min=float(pr.lambda_min), lambda_max=float(pr.lambda_max),
                 screen_pass=bool(S.bf16_screen(pr)))
        out[f"{vf}_{p}"] = d
        print(N, vf, p, pr.kappa_eff, rep.iterations, rep.converged,
              f"{time.time() - t0:.1f}s", flush=True)
    return out


def big(S, N):
    """configs[3] at N=100 (or the 80^3 size): uniform rho=0.5, p=3."""
    g, op = _problem(S, N, 0.5, 3.0, kind="uniform")
    n = op.n_free
    idx = np.unique(np.linspace(0, n - 1, N_SAMPLE).astype(np.int64))
    out = {"n_free": n, "idx": idx.tolist()}
    u = S.SplitMix64(3).gaussian(n)
    y16 = op.matvec_tagged(u.astype(np.float32), S.PrecisionTag.BF16EMU)
    y32 = op.matvec_tagged(u.astype(np.float32), S.PrecisionTag.FP32)
    y64 = op.matvec_tagged(u, S.PrecisionTag.FP64)
    for k, y in (("y16", y16), ("y32", y32), ("y64", y64)):
        y = np.asarray(y, dtype=np.float64)
        out[k] = y[idx].tolist()
        out[k + "_norm"] = float(np.linalg.norm(y))
        out[k + "_dot_u"] = float(np.dot(y, u))
    t0 = time.time()
    h = _hier(S, op, "fp32")
    out["setup_s"] = time.time() - t0
    out["lams"] = [float(lev.lam_max) for lev in h.levels]
    out["nfree"] = [int(lev.n_free) for lev in h.levels]
    out["coarsest_mode"] = h.coarsest.mode
    out["coarsest_eps"] = float(h.coarsest.eps)
    r = S.SplitMix64(7).gaussian(n)
    z = h.vcycle(r)
    out["vcycle"] = z[idx].tolist()
    out["vcycle_norm"] = float(np.linalg.norm(z))
    out["vcycle_dot_r"] = float(np.dot(z, r))
    rep = S.pcg(op.matvec, h.vcycle, g.load[g.free_dofs], S.SolverConfig(tol=1e-6, maxiter=200))
    out["pcg"] = _rep(rep)
    out["pcg"]["wall_time"] = rep.wall_time
    out["compliance"] = float(op.compliance(rep.x))
    print(N, rep.iterations, rep.final_true_residual, flush=True)
    return out


def main(argv):
    sys.path.insert(0, REF)
    import simpgmg as S
    kind, N = argv[0], int(argv[1])
    if kind == "fp32":
        res, name = fp32(S, N), f"sweep_fp32_{N}.json"
    elif kind == "jacobi":
        res, name = jacobi(S, N), f"sweep_jacobi_{N}.json"
    elif kind == "bf16":
        lo, hi = (int(v) for v in argv[2].split("-"))
        res, name = bf16(S, N, range(lo, hi + 1)), f"sweep_bf16_{N}_{lo}-{hi}.json"
    elif kind == "big":
        res, name = big(S, N), f"big_{N}.json"
    else:
        raise SystemExit(__doc__)
    res = {"recipe": " ".join(argv), "cores": os.cpu_count(), "cells": res}
    with open(os.path.join(OUT, name), "w", encoding="utf-8") as fh:
        json.dump(res, fh, indent=0, sort_keys=True)
        fh.write("\n")
    print("wrote", name)


if __name__ == "__main__":
    main(sys.argv[1:])
