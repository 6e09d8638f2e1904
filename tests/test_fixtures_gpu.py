"""Device fixture generators (states.py:58-111, prng.py:20-52,
bench/specs.py:23-34): sg_make_state draws each density field straight into HBM
and must equal the reference's fields bit for bit."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "contracts.npz")
KINDS = ("uniform", "binary", "checkerboard", "layered", "random_floor", "mixed_near_void")


@pytest.mark.parametrize("kind", KINDS)
def test_device_state_matches_reference_golden(kind):
    import paper_2604_26441_b200 as P
    gold = np.load(GOLDEN)[f"rho_{kind}"]       # made by the reference itself (oracle/make_golden.py)
    f = P.make_state(kind, 6, 4, 3, vf=0.4, floor=1e-2, seed=11, device=True)
    assert f.rho.is_cuda
    got = f.rho.cpu().numpy()
    assert got.dtype == np.float64 and np.array_equal(got.view(np.uint64), gold.view(np.uint64))
    assert f.label == P.make_state(kind, 6, 4, 3, vf=0.4, floor=1e-2, seed=11).label


@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("dims,seed", [((37, 23, 11), 0), ((64, 48, 40), 2**63 + 12345)])
def test_device_state_matches_host_port(kind, dims, seed):
    import paper_2604_26441_b200 as P
    host = P.make_state(kind, *dims, vf=0.37, floor=3e-3, seed=seed).rho
    dev = P.make_state(kind, *dims, vf=0.37, floor=3e-3, seed=seed, device=True).rho.cpu().numpy()
    assert np.array_equal(dev.view(np.uint64), host.view(np.uint64))


def test_robustness_cases_on_device():
    import paper_2604_26441_b200 as P
    from paper_2604_26441_b200.bench.specs import ROBUSTNESS_CASES
    for kind, vf, p, floor, seed in ROBUSTNESS_CASES:
        host = P.make_state(kind, 16, 8, 8, vf=vf, floor=floor, seed=seed)
        dev = P.make_state(kind, 16, 8, 8, vf=vf, floor=floor, seed=seed, device=True)
        assert np.array_equal(dev.rho.cpu().numpy(), host.rho), (kind, seed)
        Eh, Ed = P.simp_modulus(host, p), P.simp_modulus(dev, p)
        assert np.array_equal(Eh.E, Ed.E)


def test_operator_from_device_fixture():
    import paper_2604_26441_b200 as P
    g = P.build_cantilever(12, 6, 6)
    Eh = P.simp_modulus(P.make_state("mixed_near_void", 12, 6, 6, seed=19), 3.0)
    Ed = P.simp_modulus(P.make_state("mixed_near_void", 12, 6, 6, seed=19, device=True), 3.0)
    u = P.SplitMix64(3).gaussian(g.n_free)
    assert np.array_equal(P.FineOperator(g, Eh).matvec(u), P.FineOperator(g, Ed).matvec(u))
