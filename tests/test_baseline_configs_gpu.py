"""BASELINE.json configs on the GPU against the reference's measured results
(the reference package run on CPU, same fixtures and seeds).
Iteration counts are compared exactly (the north-star bar is +-2) and the
convergence verdicts must agree."""

import warnings

import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2604_26441_b200")

CFG = dict(tol=1e-6, maxiter=200)


def _solve(N, kind, vf, p, policy="fp32", jacobi=False):
    g = P.build_cantilever(N, N, N)
    st = P.make_state(kind, N, N, N, vf=vf, floor=1e-2, seed=42) if kind == "binary" else \
        P.make_state("uniform", N, N, N, vf=vf)
    op = P.FineOperator(g, P.simp_modulus(st, p))
    b = g.load[g.free_dofs]
    if jacobi:
        return P.flat_jacobi_pcg(op, b, P.SolverConfig(**CFG))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        h = P.build_hierarchy(op, 4, policy)
    return P.pcg(op.matvec, h.vcycle, b, P.SolverConfig(**CFG))


# (N, vf, p) -> reference iterations (None = capped at 200), SURVEY.md A.5 sweep table
SWEEP = [(60, 0.2, 1.5, 105), (60, 0.2, 3.0, None), (60, 0.5, 3.0, 33), (60, 0.8, 4.5, 13),
         (80, 0.2, 1.5, 115), (80, 0.2, 4.5, None), (80, 0.5, 1.5, 41), (80, 0.8, 3.0, 15)]


@pytest.mark.parametrize("N,vf,p,ref", SWEEP)
def test_sweep_cells_match_reference(N, vf, p, ref):
    rep = _solve(N, "binary", vf, p)
    if ref is None:
        assert not rep.converged and rep.iterations == 200 and rep.failure_kind == "cap"
    else:
        assert rep.converged and rep.iterations == ref


def test_config3_headline_100cube():
    """configs[3]: 16 iterations, FP64 true residual 5.71e-7 in the reference."""
    rep = _solve(100, "uniform", 0.5, 3.0)
    assert rep.converged and rep.iterations == 16
    assert rep.final_true_residual == pytest.approx(5.71e-7, rel=0.05)


def test_config4_200cube_single_gpu():
    """configs[4] on one GPU: 19 iterations, true residual 8.85e-7 in the reference."""
    rep = _solve(200, "uniform", 0.5, 3.0)
    assert rep.converged and rep.iterations == 19
    assert rep.final_true_residual == pytest.approx(8.85e-7, rel=0.05)


def test_config1_jacobi_pcg_caps():
    """configs[1] comparator: Jacobi-PCG hits the cap in every 60^3 sweep cell (true residuals
    0.13-10.3 in the reference); one cell here."""
    rep = _solve(60, "binary", 0.5, 3.0, jacobi=True)
    assert not rep.converged and rep.iterations == 200
    assert 0.1 < rep.final_true_residual < 11.0
