"""Every BASELINE.json config on the GPU against the REAL reference's results.

The expected values are fixtures made by running the unmodified reference package
(``oracle/make_golden_sweep.py``, /root/reference/pkg/src, CPU) on the same
fixtures and seeds; they live in tests/golden/*.json so the GPU box needs no
/root/reference.

* configs[1]/[2] FP32-GMG sweep: 27 cells (40^3 / 60^3 / 80^3 x vf {0.2,0.5,0.8} x
  p {1.5,3,4.5}, binary density, seed 42, floor 1e-2): identical verdicts,
  iterations within +-2 (north star), true residual of capped cells within 5%,
  residual histories of converged cells within max(1e-4, 5 x the reference's own
  rounding-noise band) per entry (``_check_history``; bands from
  oracle/make_noise_bands.py).
* configs[1] comparator: Jacobi-PCG on the nine 60^3 cells, all capped at 200.
* configs[2] guarded BF16-GMG at 80^3 (bench/runner.py:319-343 cell recipe): Lanczos
  kappa_eff within 1e-5, same screen verdict, same FGMRES(50) verdict, iterations +-2.
* configs[3] 100^3 headline and the 80^3 size: BF16 / FP32 / FP64 fine applies at
  4096 strided entries + norms, hierarchy shape and lambda_max, a V-cycle (which runs
  the production 147-brick pcg80 coarsest solve at 100^3), PCG history within the
  band rule above (the oracle's own band at 100^3 reaches 8e-3 at entry 12),
  iterations, true residual.
"""

import json
import os
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2604_26441_b200")

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CFG = dict(tol=1e-6, maxiter=200)
VFS = (0.2, 0.5, 0.8)
PS = (1.5, 3.0, 4.5)


def _gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)["cells"]


def _bf16_gold():
    out = {}
    for f in sorted(os.listdir(GOLD)):
        if f.startswith("sweep_bf16_80_"):
            out.update(_gold(f))
    return out


def _problem(N, vf, p, kind="binary"):
    g = P.build_cantilever(N, N, N)
    st = (P.make_state("binary", N, N, N, vf=vf, floor=1e-2, seed=42) if kind == "binary"
          else P.make_state("uniform", N, N, N, vf=vf))
    return g, P.FineOperator(g, P.simp_modulus(st, p))


def _hier(op, policy):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return P.build_hierarchy(op, 4, policy)


# Rounding-noise bands of the reference's own histories (oracle/make_noise_bands.py):
# per entry, the relative distance between the oracle's history and the oracle's
# history with one legitimate change of rounding order (FP32 apply accumulated in
# FP64; FP64 contraction by einsum instead of dgemm).  A history is accepted when
# every entry is within max(1e-4, BAND_K x envelope) of the reference's; the envelope
# at entry i is the largest band at that entry over the cells of the same grid size.
BAND_K = 5.0


def _band_env(name, n, cells=None):
    with open(os.path.join(GOLD, name)) as fh:
        d = json.load(fh)["cells"]
    bands = [np.asarray(v["band"]) for k, v in d.items() if cells is None or k in cells]
    bands = [b for b in bands if len(b)]
    return np.array([max(b[min(i, len(b) - 1)] for b in bands) for i in range(n)])


def _check_history(hist, ref_hist, env=None, floor=1e-4):
    n = min(len(hist), len(ref_hist))
    h = np.asarray(hist[:n])
    r = np.asarray(ref_hist[:n])
    rel = np.abs(h - r) / np.abs(r)
    tol = np.full(n, floor) if env is None else np.maximum(floor, BAND_K * np.asarray(env[:n]))
    if os.environ.get("SG_HIST_REPORT"):
        print(f"HIST n={n} maxrel={rel.max():.3e} at {int(rel.argmax())} "
              f"worst ratio to tol {float((rel / tol).max()):.3f}")
        return
    bad = rel > tol
    assert not bad.any(), (int(np.argmax(bad)), float(rel[np.argmax(bad)]),
                           float(tol[np.argmax(bad)]))


SWEEP = [(N, vf, p) for N in (40, 60, 80) for vf in VFS for p in PS]


@pytest.mark.parametrize("N,vf,p", SWEEP)
def test_fp32_sweep_cell_matches_reference(N, vf, p):
    ref = _gold(f"sweep_fp32_{N}.json")[f"{vf}_{p}"]
    g, op = _problem(N, vf, p)
    rep = P.pcg(op.matvec, _hier(op, "fp32").vcycle, g.load[g.free_dofs], P.SolverConfig(**CFG))
    assert rep.converged == ref["converged"]
    assert rep.failure_kind == ref["failure_kind"]
    assert abs(rep.iterations - ref["iterations"]) <= 2, (rep.iterations, ref["iterations"])
    if ref["converged"]:
        assert rep.final_true_residual < 1e-6
        if rep.iterations == ref["iterations"]:
            _check_history(rep.residual_history, ref["residual_history"],
                           _band_env(f"band_fp32_{N}.json", rep.iterations))
    else:
        assert rep.final_true_residual == pytest.approx(ref["final_true_residual"], rel=0.05)


@pytest.mark.parametrize("vf,p", [(vf, p) for vf in VFS for p in PS])
def test_jacobi_pcg_comparator_60cube_caps(vf, p):
    """configs[1] comparator: flat Jacobi-PCG hits the 200 cap in all nine 60^3 cells
    (PAPER.md:1037-1041), with the reference's true residual."""
    ref = _gold("sweep_jacobi_60.json")[f"{vf}_{p}"]
    g, op = _problem(60, vf, p)
    rep = P.flat_jacobi_pcg(op, g.load[g.free_dofs], P.SolverConfig(**CFG))
    assert not ref["converged"] and ref["iterations"] == 200
    assert not rep.converged and rep.iterations == 200 and rep.failure_kind == "cap"
    # 200 unpreconditioned-by-multigrid CG steps on a 1e8-contrast field: the oracle's
    # own rounding band reaches 4e-3 by step 50 (band_jacobi_60.json), and the true
    # residual at the cap moves by a few percent (north star: within 2x)
    assert rep.final_true_residual == pytest.approx(ref["final_true_residual"], rel=0.1)
    _check_history(rep.residual_history[:50], ref["residual_history"][:50],
                   _band_env("band_jacobi_60.json", 50), floor=1e-6)


@pytest.mark.parametrize("vf,p", [(vf, p) for vf in VFS for p in PS])
def test_bf16_guarded_cell_80cube(vf, p):
    """configs[2]: FP64-hierarchy Lanczos probe -> eps*kappa screen, then FGMRES(50),
    cap 500 on the BF16 hierarchy (bench/runner.py:319-343)."""
    ref = _bf16_gold().get(f"{vf}_{p}")
    if ref is None:
        pytest.skip("reference fixture for this cell not generated")
    g, op = _problem(80, vf, p)
    h64 = _hier(op, "fp64")
    probe = P.lanczos_kappa_eff(P.PreconditionedOperator(op, h64), g.n_free, 40, 0)
    assert probe.kappa_eff == pytest.approx(ref["kappa_eff"], rel=1e-5)
    assert P.bf16_screen(probe) == ref["screen_pass"]
    h16 = _hier(op, "bf16")
    rep = P.fgmres(op.matvec, h16.vcycle, g.load[g.free_dofs],
                   P.SolverConfig(method="fgmres", tol=1e-6, maxiter=500, restart=50))
    assert rep.converged == ref["converged"]
    assert abs(rep.iterations - ref["iterations"]) <= 2, (rep.iterations, ref["iterations"])
    if not ref["converged"]:
        assert rep.final_true_residual == pytest.approx(ref["final_true_residual"], rel=0.1)


@pytest.fixture(scope="module", params=[80, 100])
def big(request):
    N = request.param
    ref = _gold(f"big_{N}.json")
    g, op = _problem(N, 0.5, 3.0, kind="uniform")
    return N, ref, g, op


def test_big_fine_applies_match_reference(big):
    """BF16 (tcgen05, z-chunked multi-tile at these sizes), FP32 and FP64 applies."""
    N, ref, g, op = big
    idx = np.asarray(ref["idx"])
    u = P.SplitMix64(3).gaussian(g.n_free)
    ys = {"y16": op.matvec_tagged(u.astype(np.float32), P.PrecisionTag.BF16EMU),
          "y32": op.matvec_tagged(u.astype(np.float32), P.PrecisionTag.FP32),
          "y64": op.matvec_tagged(u, P.PrecisionTag.FP64)}
    for key, tol in (("y16", 1e-6), ("y32", 1e-6), ("y64", 1e-13)):
        y = np.asarray(ys[key], np.float64)
        yr = np.asarray(ref[key])
        scale = np.abs(yr).max()
        # per sampled entry, relative to the vector's scale (FP32 accumulation order
        # differs from OpenBLAS sgemm + np.add.at)
        assert np.abs(y[idx] - yr).max() <= (40 * tol) * scale, key
        assert np.linalg.norm(y) == pytest.approx(ref[key + "_norm"], rel=tol), key
        assert float(np.dot(y, u)) == pytest.approx(ref[key + "_dot_u"], rel=10 * tol), key


def test_big_hierarchy_vcycle_and_pcg_match_reference(big):
    N, ref, g, op = big
    h = _hier(op, "fp32")
    assert [lev.n_free for lev in h.levels] == ref["nfree"]
    assert h.coarsest.mode == ref["coarsest_mode"]
    assert h.coarsest.eps == pytest.approx(ref["coarsest_eps"], rel=1e-12)
    np.testing.assert_allclose([lev.lam_max for lev in h.levels], ref["lams"], rtol=1e-10)
    idx = np.asarray(ref["idx"])
    r = P.SplitMix64(7).gaussian(g.n_free)
    z = h.vcycle(r)
    zr = np.asarray(ref["vcycle"])
    # FP32-policy V-cycle: level 0 in FP32 (tolerance as tests/test_gpu_parity.py)
    assert np.abs(z[idx] - zr).max() <= 2e-5 * np.abs(zr).max()
    assert np.linalg.norm(z) == pytest.approx(ref["vcycle_norm"], rel=2e-5)
    assert float(np.dot(z, r)) == pytest.approx(ref["vcycle_dot_r"], rel=2e-5)
    rep = P.pcg(op.matvec, h.vcycle, g.load[g.free_dofs], P.SolverConfig(**CFG))
    rr = ref["pcg"]
    assert rep.converged and rr["converged"]
    assert rep.iterations == rr["iterations"]
    _check_history(rep.residual_history, rr["residual_history"],
                   _band_env(f"band_big_{N}.json", rep.iterations))
    assert rep.final_true_residual == pytest.approx(rr["final_true_residual"], rel=0.05)
    assert op.compliance(rep.x) == pytest.approx(ref["compliance"], rel=1e-6)


def test_config4_200cube_single_gpu():
    """configs[4] on one GPU: 19 iterations, true residual 8.85e-7 in the reference
    (311.8 s on 8 CPU cores)."""
    g, op = _problem(200, 0.5, 3.0, kind="uniform")
    rep = P.pcg(op.matvec, _hier(op, "fp32").vcycle, g.load[g.free_dofs], P.SolverConfig(**CFG))
    assert rep.converged and rep.iterations == 19
    assert rep.final_true_residual == pytest.approx(8.85e-7, rel=0.05)
