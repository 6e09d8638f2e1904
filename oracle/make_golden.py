"""Generate the golden fixtures in tests/golden/ by running the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py          # .npz vectors
    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py bench    # bench_reports.json

It imports ``simpgmg`` from /root/reference/pkg/src (read-only) and writes
small .npz files.  ``tests/test_oracle_golden.py`` pins ``oracle/simp_oracle.py``
against these vectors; the GPU parity tests then compare the sm_100a product
against the oracle on the GPU box, where /root/reference does not exist.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")


def _csr(prefix, A, out):
    out[prefix + "_indptr"] = A.indptr.astype(np.int64)
    out[prefix + "_indices"] = A.indices.astype(np.int64)
    out[prefix + "_data"] = A.data


def main():
    sys.path.insert(0, REF)
    import simpgmg as S
    from simpgmg.transfer import local_prolongation_patterns

    os.makedirs(OUT, exist_ok=True)

    # --- L0 contracts: element, prng, states, bf16 -------------------------
    out = {}
    out["ke"] = S.unit_element_stiffness(0.3).ke
    out["ke_nu0"] = S.unit_element_stiffness(0.0).ke
    for seed in (0, 1, 42, 2**63 + 5):
        g = S.SplitMix64(seed)
        out[f"u64_{seed}"] = g.next_u64(17)
        out[f"gauss_{seed}"] = S.SplitMix64(seed).gaussian(33)
    from simpgmg.prng import gaussian_unit_vector
    out["unit_1001_3"] = gaussian_unit_vector(1001, 3)
    for kind in ("uniform", "binary", "checkerboard", "layered", "random_floor",
                 "mixed_near_void"):
        out[f"rho_{kind}"] = S.make_state(kind, 6, 4, 3, vf=0.4, floor=1e-2, seed=11).rho
    out["E_binary_p3"] = S.simp_modulus(S.make_state("binary", 6, 4, 3, vf=0.5, seed=42), 3.0).E
    xs = np.array([0.1, 1.0, -2.5, 3.4e38, 1e-40, np.inf, -np.inf, 65504.0, 1.00390625,
                   1.01171875], dtype=np.float32)
    bits = np.array([0x3F808000, 0x3F818000, 0x7F7FFFFF, 0x00000001], dtype=np.uint32)
    xs = np.concatenate([xs, bits.view(np.float32),
                         S.SplitMix64(5).gaussian(1000).astype(np.float32)])
    out["bf16_in"] = xs
    out["bf16_out"] = S.round_bf16(xs)
    out["patterns"] = local_prolongation_patterns()
    np.savez_compressed(os.path.join(OUT, "contracts.npz"), **out)

    # --- fine operator ------------------------------------------------------
    out = {}
    for tag_dims, state in (((4, 2, 2), "uniform"), ((6, 4, 2), "binary"), ((5, 3, 4), "random_floor")):
        key = "x".join(map(str, tag_dims)) + "_" + state
        g = S.build_cantilever(*tag_dims)
        op = S.FineOperator(g, S.simp_modulus(S.make_state(state, *tag_dims, vf=0.5, seed=42)))
        u = S.SplitMix64(3).gaussian(g.n_free)
        out[key + "_E"] = op.modulus.E
        out[key + "_u"] = u
        out[key + "_y64"] = op.matvec_tagged(u, S.PrecisionTag.FP64)
        out[key + "_y32"] = op.matvec_tagged(u.astype(np.float32), S.PrecisionTag.FP32)
        out[key + "_y16"] = op.matvec_tagged(u.astype(np.float32), S.PrecisionTag.BF16EMU)
        out[key + "_diag"] = op.diagonal()
        out[key + "_load"] = g.load[g.free_dofs]
    # diagonal floor case (test_fine_operator.py:99-115 style)
    g = S.build_cantilever(1, 2, 1)
    op = S.FineOperator(g, S.simp_modulus(S.make_state("layered", 1, 2, 1, floor=0.0),
                                          p=1.0, emin=1e-30, e0=1.0))
    out["floor_diag"] = op.diagonal()
    np.savez_compressed(os.path.join(OUT, "fine.npz"), **out)

    # --- transfers and Galerkin operators ----------------------------------
    out = {}
    cases = (((8, 4, 4), "uniform"), ((8, 4, 4), "binary"), ((16, 8, 8), "uniform"),
             ((12, 8, 4), "random_floor"), ((16, 16, 16), "binary"))
    for dims, state in cases:
        key = "x".join(map(str, dims)) + "_" + state
        g = S.build_cantilever(*dims)
        op = S.FineOperator(g, S.simp_modulus(S.make_state(state, *dims, vf=0.5, seed=42)))
        t0 = S.build_transfer(g)
        K1 = S.assemble_level1(op, t0)
        _csr(key + "_P0", t0.P, out)
        _csr(key + "_K1", K1, out)
        try:
            t1 = S.build_transfer(t0.coarse)
            _csr(key + "_K2", S.triple_product(t1.P, K1), out)
        except S.CoarseningUnavailableError:
            pass
    np.savez_compressed(os.path.join(OUT, "galerkin.npz"), **out)

    # --- hierarchies, cycles, solvers --------------------------------------
    out = {}
    for dims, state, policy in (((8, 4, 4), "uniform", "fp64"), ((8, 4, 4), "uniform", "fp32"),
                                ((8, 4, 4), "binary", "bf16"), ((16, 8, 8), "uniform", "fp32"),
                                ((16, 8, 8), "binary", "fp32")):
        key = "x".join(map(str, dims)) + f"_{state}_{policy}"
        g = S.build_cantilever(*dims)
        op = S.FineOperator(g, S.simp_modulus(S.make_state(state, *dims, vf=0.5, seed=42)))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            h = S.build_hierarchy(op, 4, policy)
        out[key + "_lams"] = np.array([lev.lam_max for lev in h.levels])
        out[key + "_nfree"] = np.array([lev.n_free for lev in h.levels])
        out[key + "_eps"] = np.array([h.coarsest.eps])
        out[key + "_mode"] = np.array([h.coarsest.mode == "dense_cholesky"])
        r = S.SplitMix64(7).gaussian(g.n_free)
        out[key + "_r"] = r
        out[key + "_vcycle"] = h.vcycle(r)
        b = g.load[g.free_dofs]
        method = "fgmres" if policy == "bf16" else "pcg"
        cfg = S.SolverConfig(method=method, tol=1e-6, maxiter=200)
        rep = (S.pcg if method == "pcg" else S.fgmres)(op.matvec, h.vcycle, b, cfg)
        out[key + "_hist"] = np.array(rep.residual_history)
        out[key + "_iters"] = np.array([rep.iterations])
        out[key + "_conv"] = np.array([rep.converged])
        out[key + "_true"] = np.array([rep.final_true_residual])
        out[key + "_x"] = rep.x
    # forced pcg80 coarsest (test_hierarchy.py:151-158)
    g = S.build_cantilever(8, 4, 4)
    op = S.FineOperator(g, S.simp_modulus(S.make_state("uniform", 8, 4, 4, vf=0.5)))
    h = S.build_hierarchy(op, 3, "fp64", cholesky_cutoff=0)
    r = S.SplitMix64(9).gaussian(g.n_free)
    out["pcg80_vcycle"] = h.vcycle(r)
    out["pcg80_r"] = r
    # flat Jacobi baseline
    rep = S.flat_jacobi_pcg(op, g.load[g.free_dofs], S.SolverConfig(tol=1e-6, maxiter=200))
    out["jacobi_hist"] = np.array(rep.residual_history)
    out["jacobi_iters"] = np.array([rep.iterations])
    # Lanczos probe
    h64 = S.build_hierarchy(op, 3, "fp64")
    pr = S.lanczos_kappa_eff(lambda v: h64.vcycle(op.matvec(v)), g.n_free, 20, 0)
    out["lanczos"] = np.array([pr.kappa_eff, pr.lambda_min, pr.lambda_max])
    np.savez_compressed(os.path.join(OUT, "solvers.npz"), **out)

    # --- one BASELINE config-1 point: 40^3 uniform FP32-GMG PCG -------------
    out = {}
    g = S.build_cantilever(40, 40, 40)
    op = S.FineOperator(g, S.simp_modulus(S.make_state("uniform", 40, 40, 40, vf=0.5), 3.0))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = S.build_hierarchy(op, 4, "fp32")
    rep = S.pcg(op.matvec, h.vcycle, g.load[g.free_dofs], S.SolverConfig(tol=1e-6, maxiter=200))
    out["lams"] = np.array([lev.lam_max for lev in h.levels])
    out["nfree"] = np.array([lev.n_free for lev in h.levels])
    out["nnz"] = np.array([0] + [lev.operator.nnz for lev in h.levels[1:]])
    out["hist"] = np.array(rep.residual_history)
    out["iters"] = np.array([rep.iterations])
    out["true"] = np.array([rep.final_true_residual])
    out["compliance"] = np.array([op.compliance(rep.x)])
    np.savez_compressed(os.path.join(OUT, "cfg40.npz"), **out)
    print("wrote", sorted(os.listdir(OUT)))


# Specs whose reference reports pin the GPU-backed bench layer
# (tests/test_bench_layer_*.py): overrides on top of the ExperimentSpec defaults.
BENCH_SPECS = {
    "validate": {"experiment": "validate"},
    "solve": {"experiment": "solve", "grid": (16, 8, 8), "trials": 2, "warmups": 1},
    "probe": {"experiment": "probe"},
    "sweep": {"experiment": "sweep"},
    "sweep_precisions": {"experiment": "sweep", "grids": ((8, 4, 4),), "vfs": (0.5,),
                         "ps": (3.0,), "precisions": ("fp64", "fp32", "bf16"),
                         "smoothers": ("chebyshev", "jacobi")},
    "robustness": {"experiment": "robustness", "restart": 50, "maxiter": 500},
    "sweep_axes": {"experiment": "sweep", "grids": ((8, 4, 4),), "vfs": (0.5,), "ps": (3.0,),
                   "degrees": (2, 3), "depths": (2, 3), "restarts": (16, 32),
                   "precisions": ("bf16",)},
    "solve_jacobi": {"experiment": "solve", "grid": (8, 4, 4), "method": "jacobi", "trials": 1,
                     "warmups": 0, "state": "binary"},
    "probe_layered": {"experiment": "probe", "grid": (8, 4, 4), "state": "layered", "p": 4.5},
}


def bench_reports():
    """Reference numeric payloads (wall-clock fields stripped) -> bench_reports.json."""
    import json
    from dataclasses import replace
    sys.path.insert(0, REF)
    from simpgmg.bench import reports, runner, specs
    out = {}
    for name, over in BENCH_SPECS.items():
        spec = replace(specs.ExperimentSpec(), **over)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = runner.run_experiment(spec)
        out[name] = {"overrides": json.loads(json.dumps(over)),
                     "payload": reports.numeric_payload(rep),
                     "exit_code": runner.exit_code(rep)}
    with open(os.path.join(OUT, "bench_reports.json"), "w", encoding="utf-8") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print("wrote bench_reports.json")


if __name__ == "__main__":
    if sys.argv[1:] == ["bench"]:
        bench_reports()
    else:
        main()
