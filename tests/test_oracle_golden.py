"""Pin the CPU oracle (oracle/simp_oracle.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by oracle/make_golden.py running
the real reference package (simpgmg) in the build container.  Bit-exact where
the reference is deterministic integer / ordered-FP64 work (element matrix,
PRNG, states, BF16 rounding, transfer P, level-1 / level-2 Galerkin operators,
diagonals); iteration counts and residual histories for the solvers.
"""

import os
import warnings

import numpy as np
import pytest

from oracle import simp_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name))


def test_contracts_bit_exact():
    z = _load("contracts.npz")
    assert np.array_equal(O.element_ke(0.3), z["ke"])
    assert np.array_equal(O.element_ke(0.0), z["ke_nu0"])
    assert O.element_ke(0.3)[0, 0] == pytest.approx(55.0 / 234.0, rel=1e-15)
    for seed in (0, 1, 42, 2**63 + 5):
        assert np.array_equal(O.Stream(seed).raw(17), z[f"u64_{seed}"])
        assert np.array_equal(O.Stream(seed).gauss(33), z[f"gauss_{seed}"])
    assert np.array_equal(O.unit_gauss(1001, 3), z["unit_1001_3"])
    for kind in ("uniform", "binary", "checkerboard", "layered", "random_floor",
                 "mixed_near_void"):
        assert np.array_equal(O.density(kind, 6, 4, 3, vf=0.4, floor=1e-2, seed=11),
                              z[f"rho_{kind}"])
    assert np.array_equal(O.simp(O.density("binary", 6, 4, 3, vf=0.5, seed=42), 3.0),
                          z["E_binary_p3"])
    got = O.bf16(z["bf16_in"])
    want = z["bf16_out"]
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert np.array_equal(O.child_patterns(), z["patterns"])


@pytest.mark.parametrize("dims,state", [((4, 2, 2), "uniform"), ((6, 4, 2), "binary"),
                                        ((5, 3, 4), "random_floor")])
def test_fine_operator(dims, state):
    z = _load("fine.npz")
    key = "x".join(map(str, dims)) + "_" + state
    g = O.cantilever(*dims)
    E = O.simp(O.density(state, *dims, vf=0.5, seed=42))
    ke = O.element_ke()
    assert np.array_equal(E, z[key + "_E"])
    u = z[key + "_u"]
    assert np.array_equal(g.load[g.free], z[key + "_load"])
    assert np.array_equal(O.fine_apply(g, E, ke, u, "fp64"), z[key + "_y64"])
    assert np.array_equal(O.fine_apply(g, E, ke, u.astype(np.float32), "fp32"), z[key + "_y32"])
    assert np.array_equal(O.fine_apply(g, E, ke, u.astype(np.float32), "bf16"), z[key + "_y16"])
    assert np.array_equal(O.fine_diag(g, E, ke), z[key + "_diag"])


def test_diag_floor():
    z = _load("fine.npz")
    g = O.cantilever(1, 2, 1)
    E = O.simp(O.density("layered", 1, 2, 1, floor=0.0), p=1.0, emin=1e-30, e0=1.0)
    assert np.array_equal(O.fine_diag(g, E, O.element_ke()), z["floor_diag"])


@pytest.mark.parametrize("dims,state", [((8, 4, 4), "uniform"), ((8, 4, 4), "binary"),
                                        ((16, 8, 8), "uniform"), ((12, 8, 4), "random_floor"),
                                        ((16, 16, 16), "binary")])
def test_galerkin_bit_exact(dims, state):
    z = _load("galerkin.npz")
    key = "x".join(map(str, dims)) + "_" + state
    g = O.cantilever(*dims)
    E = O.simp(O.density(state, *dims, vf=0.5, seed=42))
    ke = O.element_ke()
    P0, c1 = O.transfer(g)
    K1 = O.galerkin_l1(g, E, ke, c1)
    for name, A in (("P0", P0), ("K1", K1)):
        assert np.array_equal(A.indptr, z[f"{key}_{name}_indptr"])
        assert np.array_equal(A.indices, z[f"{key}_{name}_indices"])
        assert np.array_equal(A.data, z[f"{key}_{name}_data"])
    if f"{key}_K2_data" in z:
        P1, _ = O.transfer(c1)
        K2 = O.galerkin_next(P1, K1)
        assert np.array_equal(K2.indptr, z[f"{key}_K2_indptr"])
        assert np.array_equal(K2.indices, z[f"{key}_K2_indices"])
        assert np.array_equal(K2.data, z[f"{key}_K2_data"])


@pytest.mark.parametrize("dims,state,policy", [((8, 4, 4), "uniform", "fp64"),
                                               ((8, 4, 4), "uniform", "fp32"),
                                               ((8, 4, 4), "binary", "bf16"),
                                               ((16, 8, 8), "uniform", "fp32"),
                                               ((16, 8, 8), "binary", "fp32")])
def test_hierarchy_and_solve(dims, state, policy):
    z = _load("solvers.npz")
    key = "x".join(map(str, dims)) + f"_{state}_{policy}"
    g = O.cantilever(*dims)
    E = O.simp(O.density(state, *dims, vf=0.5, seed=42))
    ke = O.element_ke()
    h = O.Hier(g, E, ke, 4, policy)
    assert np.array_equal([lev.n for lev in h.levels], z[key + "_nfree"])
    np.testing.assert_allclose([lev.lam for lev in h.levels], z[key + "_lams"], rtol=1e-12)
    assert h.eps == pytest.approx(float(z[key + "_eps"][0]), rel=1e-14)
    assert (h.mode == "dense_cholesky") == bool(z[key + "_mode"][0])
    v = h.vcycle(z[key + "_r"])
    np.testing.assert_allclose(v, z[key + "_vcycle"], rtol=1e-9, atol=1e-12 * np.abs(v).max())
    b = g.load[g.free]
    K = lambda x: O.fine_apply(g, E, ke, x, "fp64")
    rep = (O.pcg if policy != "bf16" else O.fgmres)(K, h.vcycle, b, 1e-6, 200)
    assert rep.iterations == int(z[key + "_iters"][0])
    assert rep.converged == bool(z[key + "_conv"][0])
    np.testing.assert_allclose(rep.residual_history, z[key + "_hist"], rtol=1e-6)


def test_pcg80_jacobi_lanczos():
    z = _load("solvers.npz")
    g = O.cantilever(8, 4, 4)
    E = O.simp(O.density("uniform", 8, 4, 4, vf=0.5))
    ke = O.element_ke()
    h = O.Hier(g, E, ke, 3, "fp64", cutoff=0)
    assert h.mode == "pcg80"
    np.testing.assert_allclose(h.vcycle(z["pcg80_r"]), z["pcg80_vcycle"], rtol=1e-9, atol=1e-14)
    rep = O.jacobi_pcg(g, E, ke, g.load[g.free])
    assert rep.iterations == int(z["jacobi_iters"][0])
    np.testing.assert_allclose(rep.residual_history, z["jacobi_hist"], rtol=1e-8)
    h64 = O.Hier(g, E, ke, 3, "fp64")
    pr = O.lanczos_kappa(lambda v: h64.vcycle(O.fine_apply(g, E, ke, v)), g.n_free, 20, 0)
    np.testing.assert_allclose([pr.kappa_eff, pr.lambda_min, pr.lambda_max], z["lanczos"],
                               rtol=1e-8)


def test_config1_40cube_fp32_gmg():
    """BASELINE configs[0]: 40^3 uniform rho=0.5 p=3 cantilever, FP32-GMG PCG."""
    z = _load("cfg40.npz")
    g, E, ke = O.problem(40, 40, 40)
    rep, h = O.solve(g, E, ke, "fp32")
    assert rep.iterations == int(z["iters"][0]) == 11
    assert [lev.n for lev in h.levels] == list(z["nfree"])
    assert [0] + [lev.K.nnz for lev in h.levels[1:]] == list(z["nnz"])
    np.testing.assert_allclose([lev.lam for lev in h.levels], z["lams"], rtol=1e-12)
    np.testing.assert_allclose(rep.residual_history, z["hist"], rtol=1e-6)
