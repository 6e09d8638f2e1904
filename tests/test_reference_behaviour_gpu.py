"""The reference package's behavioural contracts, exercised through this
package's drop-in API on the B200 (every compute call goes through the C ABI).

Mirrors the properties checked by the reference's own suite
(/root/reference/pkg/tests: fine operator, transfers, smoothers, hierarchy,
krylov, diagnostics, precision) -- dense oracles, exact scalings, bit-exact
identities, convergence contracts -- restated for this implementation.
"""

import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2604_26441_b200")
sp = pytest.importorskip("scipy.sparse")

ALPHA = 1.0 / 30.0


def _op(dims, kind="uniform", vf=0.5, p=3.0, seed=0, **kw):
    g = P.build_cantilever(*dims)
    return g, P.FineOperator(g, P.simp_modulus(P.make_state(kind, *dims, vf=vf, seed=seed), p, **kw))


def _free(dims, e0=1.0):
    nx, ny, nz = dims
    g = P.make_grid(nx, ny, nz, np.zeros(3 * (nx + 1) * (ny + 1) * (nz + 1), dtype=bool))
    f = P.simp_modulus(P.make_state("uniform", nx, ny, nz, vf=0.5), p=1.0, emin=1e-12, e0=e0)
    return g, P.FineOperator(g, f)


def _hier(op, *a, **k):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return P.build_hierarchy(op, *a, **k)


# ------------------------------------------------------------ precision
def test_round_bf16_bits():
    assert P.round_bf16(0.1) == 0.10009765625
    lo = np.array([0x3F808000, 0x3F818000], dtype=np.uint32).view(np.float32)
    out = P.round_bf16(lo).view(np.uint32)
    assert list(out) == [0x3F800000, 0x3F820000]  # ties to even
    x = P.SplitMix64(3).gaussian(100000).astype(np.float32) * 1e3
    r = P.round_bf16(x)
    assert np.array_equal(P.round_bf16(r), r)
    assert np.all(r.view(np.uint32) & 0xFFFF == 0)
    special = P.round_bf16(np.array([np.inf, -np.inf, np.nan], dtype=np.float32))
    assert special[0] == np.inf and special[1] == -np.inf and np.isnan(special[2])


# -------------------------------------------------------- fine operator
def test_fine_operator_contracts():
    g, op = _free((1, 1, 1))
    E0 = op.modulus.E[0]
    for j in (0, 5, 23):
        e = np.zeros(24)
        e[j] = 1.0
        np.testing.assert_allclose(op.matvec(e), E0 * op.ke[:, j], rtol=0, atol=1e-15)
    np.testing.assert_allclose(op.diagonal(), E0 * np.diag(op.ke), rtol=1e-15, atol=0)

    g, op = _op((3, 2, 2))
    K = op.assemble_dense()
    gen = P.SplitMix64(9)
    u, v = gen.gaussian(g.n_free), gen.gaussian(g.n_free)
    assert np.linalg.norm(op.matvec(u) - K @ u) < 1e-12 * np.linalg.norm(K @ u)
    lhs = op.matvec(2.0 * u - 3.0 * v)
    assert np.linalg.norm(lhs - (2.0 * op.matvec(u) - 3.0 * op.matvec(v))) < 1e-12 * np.linalg.norm(lhs)
    op2 = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", 3, 2, 2, vf=0.5), e0=2.0, emin=2e-9))
    assert np.array_equal(op2.matvec(u), 2.0 * op.matvec(u))  # exact modulus scaling
    for s in range(5):
        w = P.SplitMix64(s).gaussian(g.n_free)
        assert w @ op.matvec(w) > 0.0
    np.testing.assert_allclose(op.diagonal(), np.diag(K), rtol=1e-14, atol=0)
    assert np.array_equal(op.matvec(u), op.matvec(u))

    g, op = _op((4, 2, 2), "binary", seed=42)
    K = op.assemble_dense()
    for s in range(3):
        w = P.SplitMix64(s).gaussian(g.n_free)
        assert np.linalg.norm(op.matvec(w) - K @ w) < 1e-12 * np.linalg.norm(K @ w)

    g, op = _op((4, 2, 2))
    u = P.SplitMix64(2).gaussian(g.n_free)
    ref = op.matvec_tagged(u, P.PrecisionTag.FP64)
    o32 = op.matvec_tagged(u.astype(np.float32), P.PrecisionTag.FP32)
    o16 = op.matvec_tagged(u.astype(np.float32), P.PrecisionTag.BF16EMU)
    assert o32.dtype == np.float32 and o16.dtype == np.float32
    e32 = np.linalg.norm(o32.astype(np.float64) - ref)
    e16 = np.linalg.norm(o16.astype(np.float64) - ref)
    assert e32 < 1e-5 * np.linalg.norm(ref) and e16 < 2.0**-8 * 50 * np.linalg.norm(ref)
    assert e16 > e32


def test_fine_operator_guards():
    g, op = _op((2, 1, 1))
    with pytest.raises(ValueError):
        op.matvec(np.zeros(g.n_free + 1))
    big = P.build_cantilever(40, 20, 10)
    bop = P.FineOperator(big, P.simp_modulus(P.make_state("uniform", 40, 20, 10, vf=0.5)))
    with pytest.raises(ValueError):
        bop.assemble_dense()
    with pytest.raises(ValueError):
        P.FineOperator(g, P.simp_modulus(P.make_state("uniform", 3, 1, 1, vf=0.5)))


def test_device_tensors_in_and_out():
    import torch
    g, op = _op((6, 4, 4))
    u = P.SplitMix64(1).gaussian(g.n_free)
    ud = torch.from_numpy(u).cuda()
    yd = op.matvec(ud)
    assert isinstance(yd, torch.Tensor) and yd.is_cuda
    assert np.array_equal(yd.cpu().numpy(), op.matvec(u))


def test_large_numpy_inputs_staged_and_owned():
    """numpy vectors >= 1 MB go through page-locked staging: the result equals
    the device-tensor path bit for bit, the caller's array can be reused as
    soon as the call returns, and the returned array is the caller's own."""
    import torch
    dims = (48, 40, 32)  # ~190 k free DOFs: 1.5 MB of float64
    g, op = _op(dims)
    u = P.SplitMix64(5).gaussian(g.n_free)
    assert u.nbytes >= 1 << 20
    ref = op.matvec(torch.from_numpy(u.copy()).cuda()).cpu().numpy()
    y1 = op.matvec(u)
    u[:] = 0.0  # the staged copy was taken inside the call
    y2 = op.matvec(P.SplitMix64(5).gaussian(g.n_free))
    assert np.array_equal(y1, ref) and np.array_equal(y2, ref)
    y1[:] = 1.0  # results do not alias each other
    assert np.array_equal(y2, ref)


# ------------------------------------------------------------ transfers
def test_transfer_weights_and_masks():
    nx = ny = nz = 2
    t = P.build_transfer(P.make_grid(nx, ny, nz, np.zeros(81, dtype=bool)))
    Pm = t.P
    for i, expect in [(0, {0: 1.0}), (1, {0: 0.5, 1: 0.5}), (2, {1: 1.0})]:
        row = Pm.getrow(3 * (i + 3 * 0 + 9 * 0)).toarray()[0][0::3]
        assert {c: row[c] for c in np.flatnonzero(row)} == expect
    np.testing.assert_allclose(np.asarray(Pm.sum(axis=1)).ravel(), 1.0, atol=1e-15)
    assert set(np.unique(Pm.data)) <= {1.0, 0.5, 0.25, 0.125}
    g = P.build_cantilever(4, 2, 2)
    t = P.build_transfer(g)
    c = t.coarse
    assert (c.nx, c.ny, c.nz) == (2, 1, 1)
    assert c.dirichlet_mask.sum() == 3 * (c.ny + 1) * (c.nz + 1)
    gen = P.SplitMix64(11)
    for _ in range(5):
        xc, yf = gen.gaussian(c.n_free), gen.gaussian(g.n_free)
        a, b = float(t.prolong(xc) @ yf), float(xc @ t.restrict(yf))
        assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)
    with pytest.raises(P.CoarseningUnavailableError):
        P.build_transfer(P.make_grid(3, 2, 2, np.zeros(3 * 4 * 3 * 3, dtype=bool)))
    with pytest.raises(P.CoarseningUnavailableError):
        P.build_transfer(P.build_cantilever(4, 2, 1))


def test_galerkin_contracts():
    for dims, kind in [((4, 2, 2), "uniform"), ((4, 2, 2), "binary"), ((8, 4, 4), "uniform")]:
        g, op = _op(dims, kind, seed=42)
        t = P.build_transfer(g)
        K1 = P.assemble_level1(op, t)
        Pd = t.P.toarray()
        ref = Pd.T @ op.assemble_dense() @ Pd
        assert np.linalg.norm(K1.toarray() - ref) < 1e-10 * np.linalg.norm(ref)
        assert np.linalg.eigvalsh(K1.toarray())[0] > 0.0
        assert K1.has_sorted_indices and not np.any(K1.data == 0.0)
    g, op = _op((4, 2, 2))
    t = P.build_transfer(g)
    K1 = P.assemble_level1(op, t)
    assert np.abs(K1.toarray() - K1.toarray().T).max() < 1e-12
    op2 = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", 4, 2, 2, vf=0.5), e0=2.0, emin=2e-9))
    assert np.array_equal(P.assemble_level1(op2, t).data, 2.0 * K1.data)
    # triple products on arbitrary CSR inputs
    g2, op3 = _op((2, 2, 2))
    from paper_2604_26441_b200.transfer import canonical_csr
    K = canonical_csr(sp.csr_matrix(op3.assemble_dense()))
    out = P.triple_product(sp.identity(K.shape[0], format="csr"), K)
    assert np.array_equal(out.indptr, K.indptr) and np.array_equal(out.indices, K.indices)
    assert np.array_equal(out.data, K.data)
    Ps = sp.csr_matrix(np.array([[1.0, 0.0], [0.5, 0.5], [0.0, 1.0]]))
    K3 = sp.csr_matrix(np.array([[2.0, -1.0, 0.0], [-1.0, 2.0, -1.0], [0.0, -1.0, 2.0]]))
    ref = Ps.toarray().T @ K3.toarray() @ Ps.toarray()
    np.testing.assert_allclose(P.triple_product(Ps, K3).toarray(), ref, rtol=0, atol=1e-15)
    with pytest.raises(ValueError):
        P.triple_product(sp.identity(4, format="csr"), sp.identity(3, format="csr"))
    # Galerkin chain: device SpGEMM on the exported operators == scipy's order, bit for bit
    g, op = _op((8, 4, 4))
    t0 = P.build_transfer(g)
    K1 = P.assemble_level1(op, t0)
    t1 = P.build_transfer(t0.coarse)
    K2 = P.triple_product(t1.P, K1)
    scipy_K2 = canonical_csr(t1.P.T @ (K1 @ t1.P))
    assert np.array_equal(K2.indptr, scipy_K2.indptr) and np.array_equal(K2.data, scipy_K2.data)


# ------------------------------------------------------------ smoothers
def _diag_apply(d):
    d = np.asarray(d, dtype=np.float64)
    return lambda x: d.astype(x.dtype) * x


def test_smoother_contracts():
    lam = 3.7
    d = np.array([2.0])
    out = P.chebyshev_smooth(_diag_apply(d), np.array([1.3]), None, 1.0 / d, lam, 1, ALPHA)
    assert out[0] == pytest.approx(2.0 / ((1 + ALPHA) * lam) * 1.3 / 2.0, rel=1e-15)
    # residual polynomial on a 100-eigenvalue diagonal operator (band sweep)
    ev = np.linspace(ALPHA * 2.0, 2.0, 100)
    b = np.ones(100)
    for nu in (1, 2, 3, 4):
        x = P.chebyshev_smooth(_diag_apply(ev), b, None, np.ones(100), 2.0, nu, ALPHA)
        res = np.abs(b - ev * x)
        assert res.max() <= P.chebyshev_band_bound(nu, ALPHA) + 1e-12
    # damped Jacobi on a diagonal operator is exact per mode
    x = P.jacobi_smooth(_diag_apply(ev), b, None, 1.0 / ev, 0.5, 3)
    np.testing.assert_allclose(b - ev * x, 0.125 * b, rtol=1e-12)
    with pytest.raises(ValueError):
        P.jacobi_smooth(_diag_apply(ev), b, None, 1.0 / ev, 0.7, 1)
    # lambda_max estimate vs the dense eigensolver
    g, op = _op((4, 2, 2))
    K = op.assemble_dense()
    dinv = 1.0 / op.diagonal()
    true = np.max(np.linalg.eigvals(np.diag(dinv) @ K).real)
    est = P.estimate_lambda_max(op.matvec, dinv, iters=200, seed=0)
    assert est == pytest.approx(true, rel=0.02)
    assert P.estimate_lambda_max(op.matvec, dinv, iters=200, seed=5) == pytest.approx(est, rel=0.01)
    # FP32 smoothing differs from FP64 but stays close
    r = P.SplitMix64(3).gaussian(g.n_free)
    x64 = P.chebyshev_smooth(op.matvec, r, None, dinv, true, 2, ALPHA, P.PrecisionTag.FP64)
    x32 = P.chebyshev_smooth(lambda v: op.matvec_tagged(v, P.PrecisionTag.FP32), r, None, dinv,
                             true, 2, ALPHA, P.PrecisionTag.FP32)
    assert not np.array_equal(x64, x32)
    assert np.linalg.norm(x64 - x32) < 1e-5 * np.linalg.norm(x64)


# ------------------------------------------------------------ hierarchy
def test_hierarchy_contracts():
    g, op = _op((2, 1, 1))
    h = P.build_hierarchy(op, levels=1, policy="fp64")
    assert h.n_levels == 1 and h.coarsest.mode == "dense_cholesky"
    r = P.SplitMix64(1).gaussian(g.n_free)
    ref = np.linalg.solve(op.assemble_dense() + h.coarsest.eps * np.eye(g.n_free), r)
    np.testing.assert_allclose(h.vcycle(r), ref, rtol=1e-12, atol=0)
    assert np.array_equal(h.vcycle(r), h.wcycle(r))

    g, op = _op((8, 4, 4))
    with pytest.warns(UserWarning):
        h = P.build_hierarchy(op, levels=10, policy="fp64")
    frees = [lev.n_free for lev in h.levels]
    assert h.n_levels == 3 and all(a > b for a, b in zip(frees, frees[1:]))
    assert h.coarsest.eps == max(float(h.levels[-1].diag.mean()) * 1e-8, 1e-14)
    for policy, expect in [("fp64", [P.PrecisionTag.FP64] * 3),
                           ("fp32", [P.PrecisionTag.FP32] + [P.PrecisionTag.FP64] * 2),
                           ("bf16", [P.PrecisionTag.BF16EMU, P.PrecisionTag.FP32, P.PrecisionTag.FP64])]:
        assert [lev.tag for lev in _hier(op, 3, policy).levels] == expect
    with pytest.raises(ValueError):
        P.build_hierarchy(op, 3, "fp8")
    gen = P.SplitMix64(5)
    r1, r2 = gen.gaussian(g.n_free), gen.gaussian(g.n_free)
    v1, v2 = h.vcycle(r1), h.vcycle(r2)
    s = np.linalg.norm(v1)
    assert np.linalg.norm(h.vcycle(3.0 * r1) - 3.0 * v1) < 1e-12 * s
    assert np.linalg.norm(h.vcycle(r1 + r2) - (v1 + v2)) < 1e-12 * s
    K = op.assemble_dense()
    for _ in range(5):
        e = gen.gaussian(g.n_free)
        ea = e - h.vcycle(K @ e)
        assert ea @ K @ ea < e @ K @ e
    b = g.load[g.free_dofs]
    rep = P.pcg(op.matvec, h.vcycle, b, P.SolverConfig(tol=1e-10, maxiter=200))
    xd = np.linalg.solve(K, b)
    assert rep.converged and np.linalg.norm(rep.x - xd) < 1e-8 * np.linalg.norm(xd)
    cfg = P.SolverConfig(tol=1e-6, maxiter=200)
    assert P.pcg(op.matvec, h.wcycle, b, cfg).iterations <= P.pcg(op.matvec, h.vcycle, b, cfg).iterations
    h1 = P.build_hierarchy(op, 1, "fp64")
    assert P.symmetry_defect(h1, 5, 0) < 1e-12
    d64 = P.symmetry_defect(_hier(op, 3, "fp64"), 5, 0)
    assert P.symmetry_defect(_hier(op, 3, "bf16"), 5, 0) >= d64
    hp = P.build_hierarchy(op, 3, "fp64", cholesky_cutoff=0)
    assert hp.coarsest.mode == "pcg80" and P.pcg(op.matvec, hp.vcycle, b, cfg).converged
    hs = P.build_hierarchy(op, 3, "fp64", P.SmootherConfig("jacobi", degree=3, omega=0.4),
                           coarse_smooth_steps=2)
    assert hs.levels[0].smoother.degree == 3 and hs.levels[1].smoother.degree == 2
    assert hs.levels[1].smoother.omega == 0.4


def test_wcycle_equals_hand_rolled_two_level():
    g, op = _op((4, 2, 2))
    h = P.build_hierarchy(op, 2, "fp64")
    r = P.SplitMix64(7).gaussian(g.n_free)
    lev = h.levels[0]
    t = lev.transfer
    x = lev.smooth(r, None)
    for _ in range(2):
        d = r - lev.matvec64(x)
        x = x + t.prolong(h.coarsest.solve(t.restrict(d)))
    assert np.array_equal(h.wcycle(r), lev.smooth(r, x))


def test_two_grid_exactness_and_lambda_cache():
    g, op = _op((4, 2, 2))
    t = P.build_transfer(g)
    K = op.assemble_dense()
    Pd = t.P.toarray()
    e = P.SplitMix64(2).gaussian(g.n_free)
    corr = e - Pd @ np.linalg.solve(Pd.T @ K @ Pd, Pd.T @ (K @ e))
    assert np.abs(Pd.T @ (K @ corr)).max() < 1e-10 * np.abs(Pd.T @ (K @ e)).max()
    h = P.build_hierarchy(op, 2, "fp64")
    near = P.FineOperator(g, P.simp_modulus(P.make_state("uniform", 4, 2, 2, vf=0.5), e0=1.05, emin=1e-9))
    assert [a.lam_max for a in P.build_hierarchy(near, 2, "fp64", lambda_cache=h).levels] == \
        [a.lam_max for a in h.levels]
    far = P.FineOperator(g, P.simp_modulus(P.make_state("binary", 4, 2, 2, vf=0.5, seed=3)))
    assert P.build_hierarchy(far, 2, "fp64", lambda_cache=h).levels[0].lam_max != h.levels[0].lam_max


# ---------------------------------------------------------------- krylov
def test_krylov_contracts():
    ident = lambda x: x
    b = P.SplitMix64(1).gaussian(20)
    rep = P.pcg(ident, ident, b, P.SolverConfig(tol=1e-6, maxiter=10))
    assert rep.converged and rep.iterations == 1 and rep.failure_kind == "none"
    d = np.array([1.0, 4.0, 9.0, 16.0])
    bb = np.array([2.0, -1.0, 3.0, 0.5])
    rep = P.pcg(lambda x: d * x, lambda r: r / d, bb, P.SolverConfig(tol=1e-12, maxiter=10))
    assert rep.converged and rep.iterations == 1
    np.testing.assert_allclose(rep.x, bb / d, rtol=1e-13)
    rep = P.pcg(lambda x: x * np.nan, ident, np.ones(4), P.SolverConfig(tol=1e-6, maxiter=10))
    assert not rep.converged and rep.failure_kind == "non_finite"
    rep = P.pcg(ident, ident, np.zeros(7), P.SolverConfig())
    assert rep.converged and rep.iterations == 0 and rep.final_true_residual == 0.0
    gen = P.SplitMix64(12)
    A = gen.gaussian(64).reshape(8, 8)
    K = A @ A.T + 8 * np.eye(8)
    xt = gen.gaussian(8)
    bk = K @ xt
    dk = np.diag(K)
    errs = []
    for it in range(1, 9):
        r = P.pcg(lambda v: K @ v, lambda r: r / dk, bk, P.SolverConfig(tol=1e-16, maxiter=it))
        e = r.x - xt
        errs.append(float(e @ K @ e))
    assert all(a >= c - 1e-13 * abs(a) for a, c in zip(errs, errs[1:]))

    g, op = _op((8, 4, 4))
    h = _hier(op, 3, "fp64")
    b = g.load[g.free_dofs]
    rep = P.pcg(op.matvec, h.vcycle, b, P.SolverConfig(tol=1e-6, maxiter=200))
    assert rep.converged and rep.iterations <= 30
    assert np.linalg.norm(b - op.matvec(rep.x)) < 1e-6 * np.linalg.norm(b)
    rep = P.flat_jacobi_pcg(op, b, P.SolverConfig(tol=1e-14, maxiter=5))
    assert not rep.converged and rep.failure_kind == "cap" and rep.iterations == 5
    assert len(rep.residual_history) == 5
    rep = P.flat_jacobi_pcg(op, b, P.SolverConfig(tol=1e-6, maxiter=200))
    assert rep.converged and 10 < rep.iterations < 200
    g4, op4 = _op((4, 2, 2), "binary", seed=7)
    b4 = g4.load[g4.free_dofs]
    for cfg in (P.SolverConfig(tol=1e-6, maxiter=3), P.SolverConfig(tol=1e-6, maxiter=500)):
        rep = P.flat_jacobi_pcg(op4, b4, cfg)
        tr = np.linalg.norm(b4 - op4.matvec(rep.x)) / np.linalg.norm(b4)
        assert rep.converged == (rep.final_true_residual < cfg.tol)
        assert rep.final_true_residual == pytest.approx(tr, rel=1e-12)
        if not rep.converged:
            assert rep.failure_kind == "cap" and rep.iterations == cfg.maxiter


def test_fgmres_contracts():
    ident = lambda x: x
    b = P.SplitMix64(2).gaussian(12)
    rep = P.fgmres(ident, ident, b, P.SolverConfig(method="fgmres"))
    assert rep.converged and rep.iterations == 1
    d = np.full(6, 3.0)
    e2 = np.zeros(6)
    e2[2] = 1.0
    rep = P.fgmres(lambda x: d * x, ident, e2, P.SolverConfig(method="fgmres", tol=1e-12, maxiter=50))
    assert rep.converged and rep.iterations == 1
    np.testing.assert_allclose(rep.x, e2 / 3.0, rtol=1e-14)
    gen = P.SplitMix64(4)
    A = gen.gaussian(100).reshape(10, 10)
    K = A @ A.T + 10 * np.eye(10)
    bb = gen.gaussian(10)
    rep = P.fgmres(lambda v: K @ v, lambda r: r / np.diag(K), bb,
                   P.SolverConfig(method="fgmres", tol=1e-10, maxiter=200, restart=5))
    ref = np.linalg.solve(K, bb)
    assert rep.converged and np.linalg.norm(rep.x - ref) < 1e-8 * np.linalg.norm(ref)
    gen = P.SplitMix64(8)
    A = gen.gaussian(400).reshape(20, 20)
    K = A @ A.T + 20 * np.eye(20)
    bb = gen.gaussian(20)
    rep = P.fgmres(lambda v: K @ v, ident, bb,
                   P.SolverConfig(method="fgmres", tol=1e-12, maxiter=40, restart=10))
    hh = rep.residual_history
    for start in range(0, len(hh), 10):
        cyc = hh[start:start + 10]
        assert all(a >= c - 1e-15 for a, c in zip(cyc, cyc[1:]))
    state = {"k": 0}

    def wobbly(r):
        state["k"] += 1
        return r / (np.diag(K) * (1.0 + 0.1 * (state["k"] % 3)))

    rep = P.fgmres(lambda v: K @ v, wobbly, bb, P.SolverConfig(method="fgmres", tol=1e-10,
                                                               maxiter=100, restart=6))
    assert rep.converged and np.linalg.norm(bb - K @ rep.x) < 1e-10 * np.linalg.norm(bb)
    K2 = A @ A.T + 1e-3 * np.eye(20)
    rep = P.fgmres(lambda v: K2 @ v, ident, bb, P.SolverConfig(method="fgmres", tol=1e-14,
                                                              maxiter=8, restart=4))
    assert not rep.converged and rep.failure_kind == "cap" and rep.iterations == 8
    # native FGMRES on the fine operator with a BF16 hierarchy (config-3 path)
    g, op = _op((8, 4, 4), "binary", seed=42)
    h16 = _hier(op, 4, "bf16")
    rep = P.fgmres(op.matvec, h16.vcycle, g.load[g.free_dofs],
                   P.SolverConfig(method="fgmres", tol=1e-6, maxiter=200, restart=50))
    assert rep.converged


# ----------------------------------------------------------- diagnostics
def test_lanczos_contracts():
    d = np.arange(1.0, 11.0)
    pr = P.lanczos_kappa_eff(lambda v: d * v, 10, m=10, seed=0)
    assert pr.kappa_eff == pytest.approx(10.0, abs=1e-6)
    assert pr.eps_kappa == pytest.approx(P.EPS_BF16 * pr.kappa_eff, rel=0)
    pr = P.lanczos_kappa_eff(lambda v: v.copy(), 50, m=10, seed=3)
    assert pr.kappa_eff == pytest.approx(1.0, abs=1e-8) and pr.partial
    dd = np.linspace(1.0, 5.0, 30)
    assert P.lanczos_kappa_eff(lambda v: dd * v, 30, 12, 5).kappa_eff == \
        P.lanczos_kappa_eff(lambda v: dd * v, 30, 12, 5).kappa_eff
    with pytest.raises(ValueError):
        P.lanczos_kappa_eff(lambda v: v, 10, m=1, seed=0)
    g, op = _op((8, 4, 4))
    h = _hier(op, 3, "fp64")
    native = P.lanczos_kappa_eff(P.PreconditionedOperator(op, h), g.n_free, m=40, seed=0)
    generic = P.lanczos_kappa_eff(lambda v: h.vcycle(op.matvec(v)), g.n_free, m=40, seed=0)
    assert native.kappa_eff == pytest.approx(generic.kappa_eff, rel=1e-6)
    K = op.assemble_dense()
    L = np.linalg.cholesky(K)
    n = g.n_free
    M = np.column_stack([h.vcycle(np.eye(n)[:, i]) for i in range(n)])
    S = L.T @ M @ L
    ev = np.linalg.eigvalsh(0.5 * (S + S.T))
    assert native.kappa_eff == pytest.approx(ev[-1] / ev[0], rel=0.05)
