"""CPU tests of the host-side data contracts and validators of the drop-in API.

The fixtures/constants here never touch the device: grid + DOF numbering,
splitmix64 streams, density states, the SIMP map and the element matrix must be
bit-identical to the reference (golden vectors from oracle/make_golden.py); the
config validators must raise the reference's errors.
"""

import os

import numpy as np
import pytest

import paper_2604_26441_b200 as P
from paper_2604_26441_b200.hierarchy import PRECISION_POLICIES, policy_tags

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _z(name):
    return np.load(os.path.join(GOLD, name))


def test_element_matrix_bits_and_invariants():
    ke = P.unit_element_stiffness(0.3).ke
    z = _z("contracts.npz")
    assert np.array_equal(ke, z["ke"])
    assert np.array_equal(P.unit_element_stiffness(0.0).ke, z["ke_nu0"])
    assert ke[0, 0] == pytest.approx(55.0 / 234.0, rel=1e-15)
    assert np.array_equal(ke, ke.T)
    # three rigid translations in the null space, rank 18 (6 rigid modes)
    for axis in range(3):
        t = np.zeros(24)
        t[axis::3] = 1.0
        assert np.abs(ke @ t).max() < 1e-12
    ev = np.linalg.eigvalsh(ke)
    assert np.sum(ev > 1e-10) == 18 and ev.min() > -1e-12
    with pytest.raises(ValueError):
        P.unit_element_stiffness(0.5)
    with pytest.raises(ValueError):
        P.unit_element_stiffness(-0.1)
    assert not ke.flags.writeable


def test_prng_streams_bit_exact():
    z = _z("contracts.npz")
    for seed in (0, 1, 42, 2**63 + 5):
        assert np.array_equal(P.SplitMix64(seed).next_u64(17), z[f"u64_{seed}"])
        assert np.array_equal(P.SplitMix64(seed).gaussian(33), z[f"gauss_{seed}"])
    from paper_2604_26441_b200.prng import gaussian_unit_vector
    assert np.array_equal(gaussian_unit_vector(1001, 3), z["unit_1001_3"])
    # batching independence: ten draws of one == one draw of ten
    a = P.SplitMix64(9)
    b = P.SplitMix64(9)
    assert np.array_equal(np.concatenate([a.next_u64(1) for _ in range(10)]), b.next_u64(10))
    u = P.SplitMix64(4).uniform01(100000)
    assert u.min() >= 0.0 and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01


def test_states_and_simp_bit_exact():
    z = _z("contracts.npz")
    for kind in ("uniform", "binary", "checkerboard", "layered", "random_floor", "mixed_near_void"):
        rho = P.make_state(kind, 6, 4, 3, vf=0.4, floor=1e-2, seed=11).rho
        assert np.array_equal(rho, z[f"rho_{kind}"]), kind
        assert not rho.flags.writeable
    E = P.simp_modulus(P.make_state("binary", 6, 4, 3, vf=0.5, seed=42), 3.0).E
    assert np.array_equal(E, z["E_binary_p3"])
    with pytest.raises(ValueError):
        P.make_state("sponge", 2, 2, 2)
    with pytest.raises(ValueError):
        P.make_state("binary", 2, 2, 2, vf=1.0)
    with pytest.raises(ValueError):
        P.simp_modulus(P.make_state("uniform", 2, 2, 2), p=0.0)
    with pytest.raises(ValueError):
        P.simp_modulus(P.make_state("uniform", 2, 2, 2), emin=2.0, e0=1.0)


def test_cantilever_contract():
    g = P.build_cantilever(4, 2, 3)
    assert (g.n_nodes, g.n_dof, g.n_elem) == (5 * 3 * 4, 3 * 60, 24)
    fixed_nodes = np.flatnonzero(g.dirichlet_mask[0::3])
    assert all(n % 5 == 0 for n in fixed_nodes) and len(fixed_nodes) == 12
    assert np.isclose(g.load.sum(), -1.0)
    loaded = np.flatnonzero(g.load)
    assert all(d % 3 == 1 for d in loaded)
    assert all((d // 3) % 5 == 4 and ((d // 3) // 5) % 3 == 0 for d in loaded)
    # free numbering is the sorted complement of the mask
    assert np.array_equal(g.free_dofs, np.flatnonzero(~g.dirichlet_mask))
    assert np.array_equal(g.free_map[g.free_dofs], np.arange(g.n_free))
    # element DOF table, corner order i-fastest
    e = g.element_dofs
    assert e.shape == (24, 24)
    assert list(e[0, ::3] // 3) == [0, 1, 5, 6, 15, 16, 20, 21]
    assert g.is_cantilever_mask
    with pytest.raises(ValueError):
        P.build_cantilever(0, 1, 1)
    with pytest.raises(ValueError):
        P.make_grid(1, 1, 1, np.zeros(3))
    with pytest.raises(ValueError):
        load = np.zeros(24)
        load[0] = 1.0
        mask = np.zeros(24, dtype=bool)
        mask[0] = True
        P.make_grid(1, 1, 1, mask, load)


def test_config_validation_and_bounds():
    with pytest.raises(ValueError):
        P.SolverConfig(method="bicgstab")
    with pytest.raises(ValueError):
        P.SolverConfig(tol=0.0)
    with pytest.raises(ValueError):
        P.SolverConfig(maxiter=0)
    with pytest.raises(ValueError):
        P.SolverConfig(restart=0)
    with pytest.raises(ValueError):
        P.SmootherConfig(kind="gauss-seidel")
    with pytest.raises(ValueError):
        P.SmootherConfig(degree=0)
    with pytest.raises(ValueError):
        P.SmootherConfig(omega=0.6)
    alpha = 1.0 / 30.0
    assert P.chebyshev_band_bound(2, alpha) == pytest.approx(0.778, abs=1e-3)
    assert P.chebyshev_band_bound(1, alpha) == pytest.approx(29.0 / 31.0, rel=1e-12)
    b = [P.chebyshev_band_bound(n, alpha) for n in range(1, 7)]
    assert all(x > y for x, y in zip(b, b[1:]))
    with pytest.raises(ValueError):
        P.chebyshev_band_bound(0, alpha)
    assert P.kappa_bound(0.5) == 3.0
    with pytest.raises(ValueError):
        P.kappa_bound(1.0)
    mk = lambda k: P.SpectralProbe(40, 0, k, P.EPS_BF16 * k, 0.0, 0.0, False)
    assert P.bf16_screen(mk(79.65)) and not P.bf16_screen(mk(256.0))


def test_policy_tags():
    assert policy_tags("fp32", 4) == [P.PrecisionTag.FP32] + [P.PrecisionTag.FP64] * 3
    assert policy_tags("bf16", 3) == [P.PrecisionTag.BF16EMU, P.PrecisionTag.FP32,
                                      P.PrecisionTag.FP64]
    assert set(PRECISION_POLICIES) == {"fp64", "fp32", "bf16"}
    with pytest.raises(ValueError):
        policy_tags("fp8", 2)
    assert P.PrecisionTag.FP32.working_dtype is np.float32
    assert P.PrecisionTag.FP64.working_dtype is np.float64


def test_galerkin_host_tables_match_reference_products():
    """The host constants of the level-1 aggregation are the reference's
    P_c^T Ke P_c products (transfer.py:143), evaluated with the same numpy calls."""
    from oracle import simp_oracle as O
    from paper_2604_26441_b200.hierarchy import galerkin_tables
    from paper_2604_26441_b200.transfer import local_prolongation_patterns
    ke = P.unit_element_stiffness().ke
    pats = local_prolongation_patterns()
    assert np.array_equal(pats, O.child_patterns())
    for c in range(8):
        assert np.allclose(pats[c] @ np.ones(24), np.ones(24), atol=1e-15)
    code = (2 << 24) | sum(1 << (3 * b + a) for b in range(8) if not (b & 1) for a in range(3))
    tri, diffs = galerkin_tables(ke, np.array([code], dtype=np.uint32))
    p = pats[2].copy()
    p[[3 * b + a for b in range(8) if not (b & 1) for a in range(3)]] = 0.0
    assert np.array_equal(tri[2], pats[2].T @ ke @ pats[2])
    assert np.array_equal(diffs[0], p.T @ ke @ p - tri[2])
