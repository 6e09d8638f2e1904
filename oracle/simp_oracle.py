"""CPU oracle for the PCG / geometric-multigrid hot path of arXiv 2604.26441.

TEST INFRASTRUCTURE ONLY.  This module is a numpy/scipy restatement of the
reference package ``simpgmg`` (``/root/reference/pkg/src/simpgmg``) used as
the *checker* for the sm_100a product in ``paper_2604_26441_b200``.  Only
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it; the product never
does.

Parity is pinned: ``oracle/make_golden.py`` runs the real reference in the
build container and writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks every function here against those vectors (bit-exact for integer
work, the element matrix, the level-1 / level-2 Galerkin operators and the
diagonal; iteration counts and histories for the solvers).

Each function cites the reference ``file:line`` it restates.  The numerics
deliberately use the same numpy / scipy calls as the reference so that the
rounding (OpenBLAS dgemm for the 24x24 element products, scipy sparsetools
for CSR assembly and SpGEMM, LAPACK for the dense coarsest factor) is the
same on the same host.
"""

from __future__ import annotations

import time
from types import SimpleNamespace

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

# ----------------------------------------------------------------------------
# splitmix64 stream (prng.py:26-73)

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


class Stream:
    """Counter-based splitmix64: output n is mix(seed + n*golden), n >= 1."""

    def __init__(self, seed):
        self.seed = np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF)
        self.used = 0

    def raw(self, n):
        idx = np.arange(self.used + 1, self.used + n + 1, dtype=np.uint64)
        self.used += n
        with np.errstate(over="ignore"):
            z = self.seed + _G * idx
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            return z ^ (z >> np.uint64(31))

    def u01(self, n):
        return (self.raw(n) >> np.uint64(11)).astype(np.float64) * 2.0**-53

    def gauss(self, n):
        half = (n + 1) // 2
        a = ((self.raw(half) >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
        b = self.u01(half)
        rad = np.sqrt(-2.0 * np.log(a))
        ang = 2.0 * np.pi * b
        out = np.empty(2 * half)
        out[0::2] = rad * np.cos(ang)
        out[1::2] = rad * np.sin(ang)
        return out[:n]


def unit_gauss(n, seed):
    """prng.py:57-64"""
    v = Stream(seed).gauss(n)
    s = np.linalg.norm(v)
    if s == 0.0:
        v[0], s = 1.0, 1.0
    return v / s


# ----------------------------------------------------------------------------
# grid / DOF contract (grid.py:18-123)

CORNERS = np.array([[c & 1, (c >> 1) & 1, (c >> 2) & 1] for c in range(8)],
                   dtype=np.int64)


def make_grid(nx, ny, nz, mask, load=None):
    """grid.py:64-73 (element DOFs) and :115-138 (free map)."""
    ndof = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    mask = np.asarray(mask, dtype=bool).copy()
    assert mask.shape == (ndof,)
    load = np.zeros(ndof) if load is None else np.asarray(load, np.float64).copy()
    e = np.arange(nx * ny * nz)
    ei, ej, ek = e % nx, (e // nx) % ny, e // (nx * ny)
    nodes = ((ei[:, None] + CORNERS[:, 0]) + (nx + 1) * ((ej[:, None] + CORNERS[:, 1])
             + (ny + 1) * (ek[:, None] + CORNERS[:, 2])))
    edofs = ((3 * nodes)[:, :, None] + np.arange(3)).reshape(-1, 24)
    free = np.flatnonzero(~mask)
    fmap = np.full(ndof, -1, dtype=np.int64)
    fmap[free] = np.arange(free.size)
    return SimpleNamespace(nx=nx, ny=ny, nz=nz, mask=mask, load=load, free=free,
                           fmap=fmap, edofs=edofs, n_free=free.size, n_dof=ndof,
                           n_elem=nx * ny * nz)


def cantilever(nx, ny, nz):
    """grid.py:141-162: x=0 face clamped, -1/(nz+1) on y of edge (nx, 0, k)."""
    nnode = (nx + 1) * (ny + 1) * (nz + 1)
    node = np.arange(nnode)
    mask = np.repeat(node % (nx + 1) == 0, 3)
    load = np.zeros(3 * nnode)
    edge = nx + (nx + 1) * (ny + 1) * np.arange(nz + 1)
    load[3 * edge + 1] = -1.0 / (nz + 1)
    return make_grid(nx, ny, nz, mask, load)


def node_id(g, i, j, k):
    return i + (g.nx + 1) * (j + (g.ny + 1) * k)


# ----------------------------------------------------------------------------
# density states and the SIMP map (states.py:43-111)

def density(kind, nx, ny, nz, vf=0.5, floor=1e-2, seed=0):
    n = nx * ny * nz
    e = np.arange(n)
    ei, ej, ek = e % nx, (e // nx) % ny, e // (nx * ny)
    if kind == "uniform":
        return np.full(n, float(vf))
    if kind == "binary":
        return np.where(Stream(seed).u01(n) < vf, 1.0, floor)
    if kind == "checkerboard":
        return np.where((ei + ej + ek) % 2 == 0, 1.0, floor)
    if kind == "layered":
        return np.where(2 * ej < ny, 1.0, floor)
    if kind == "random_floor":
        return floor + (1.0 - floor) * Stream(seed).u01(n)
    if kind == "mixed_near_void":
        s = Stream(seed)
        solid = s.u01(n) < vf
        demote = s.u01(n) < 0.1
        return np.where(solid & ~demote, 1.0, floor)
    raise ValueError(kind)


def simp(rho, p=3.0, emin=1e-9, e0=1.0):
    r = np.asarray(rho, dtype=np.float64)
    return emin + (e0 - emin) * r**p


# ----------------------------------------------------------------------------
# element stiffness (element.py:23-70)

def element_ke(nu=0.3):
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2.0 * mu
    D[3:, 3:] = mu * np.eye(3)
    s = 2.0 * CORNERS - 1.0
    gp = 1.0 / np.sqrt(3.0)
    ke = np.zeros((24, 24))
    for x0 in (-gp, gp):
        for x1 in (-gp, gp):
            for x2 in (-gp, gp):
                f = 1.0 + s * np.array([x0, x1, x2])
                dn = np.empty((8, 3))
                dn[:, 0] = s[:, 0] * f[:, 1] * f[:, 2]
                dn[:, 1] = f[:, 0] * s[:, 1] * f[:, 2]
                dn[:, 2] = f[:, 0] * f[:, 1] * s[:, 2]
                dn *= 2.0 / 8.0
                B = np.zeros((6, 24))
                for a in range(8):
                    B[0, 3 * a] = dn[a, 0]
                    B[1, 3 * a + 1] = dn[a, 1]
                    B[2, 3 * a + 2] = dn[a, 2]
                    B[3, 3 * a], B[3, 3 * a + 1] = dn[a, 1], dn[a, 0]
                    B[4, 3 * a + 1], B[4, 3 * a + 2] = dn[a, 2], dn[a, 1]
                    B[5, 3 * a], B[5, 3 * a + 2] = dn[a, 2], dn[a, 0]
                ke += (B.T @ D @ B) / 8.0
    return 0.5 * (ke + ke.T)


# ----------------------------------------------------------------------------
# BF16 emulation (precision.py:25-48)

def bf16(x):
    a = np.ascontiguousarray(x, dtype=np.float32)
    bits = a.view(np.uint32)
    with np.errstate(over="ignore"):
        r = (bits + np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))) \
            & np.uint32(0xFFFF0000)
    out = r.view(np.float32).copy()
    nan = np.isnan(a)
    out[nan] = a[nan]
    return out


# ----------------------------------------------------------------------------
# fine operator (fine_operator.py:53-105)

def fine_apply(g, E, ke, u, tag="fp64"):
    """fine_operator.py:56-77; modulus applied after the contraction."""
    if tag == "fp64":
        full = np.zeros(g.n_dof)
        full[g.free] = u
        loc = (full[g.edofs] @ ke) * E[:, None]
        return np.bincount(g.edofs.ravel(), weights=loc.ravel(), minlength=g.n_dof)[g.free]
    E32 = E.astype(np.float32)
    ke32 = ke.astype(np.float32)
    full = np.zeros(g.n_dof, dtype=np.float32)
    full[g.free] = u
    gat = full[g.edofs]
    if tag == "bf16":
        loc = (bf16(gat) @ bf16(ke32)) * E32[:, None]
    else:
        loc = (gat @ ke32) * E32[:, None]
    out = np.zeros(g.n_dof, dtype=np.float32)
    np.add.at(out, g.edofs.ravel(), loc.ravel())
    return out[g.free]


def fine_diag(g, E, ke):
    """fine_operator.py:79-86 (floor 1e-14 * mean)."""
    w = (E[:, None] * np.diag(ke)[None, :]).ravel()
    d = np.bincount(g.edofs.ravel(), weights=w, minlength=g.n_dof)[g.free]
    return np.maximum(d, 1e-14 * d.mean())


def fine_dense(g, E, ke):
    """fine_operator.py:88-101 (oracle assembly)."""
    K = np.zeros((g.n_free, g.n_free))
    for e in range(g.n_elem):
        idx = g.fmap[g.edofs[e]]
        keep = idx >= 0
        K[np.ix_(idx[keep], idx[keep])] += E[e] * ke[np.ix_(keep, keep)]
    return K


# ----------------------------------------------------------------------------
# transfers and Galerkin products (transfer.py:33-181)

def canon(A):
    """transfer.py:33-39"""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.eliminate_zeros()
    A.sort_indices()
    return A


def _stencil_1d(nf):
    f = np.arange(nf)
    ev, od = f[f % 2 == 0], f[f % 2 == 1]
    return (np.concatenate([ev, od, od]), np.concatenate([ev // 2, od // 2, od // 2 + 1]),
            np.concatenate([np.ones(ev.size), np.full(od.size, 0.5), np.full(od.size, 0.5)]))


def transfer(fine):
    """transfer.py:68-107 -> (P csr, coarse grid); injection mask from (2i,2j,2k)."""
    if fine.nx % 2 or fine.ny % 2 or fine.nz % 2:
        raise ValueError("odd dimension")
    cx, cy, cz = fine.nx // 2, fine.ny // 2, fine.nz // 2
    cn = np.arange((cx + 1) * (cy + 1) * (cz + 1))
    ci, cj, ck = cn % (cx + 1), (cn // (cx + 1)) % (cy + 1), cn // ((cx + 1) * (cy + 1))
    inj = node_id(fine, 2 * ci, 2 * cj, 2 * ck)
    cmask = fine.mask[(3 * inj[:, None] + np.arange(3)).ravel()]
    coarse = make_grid(cx, cy, cz, cmask)
    (fx, px, vx), (fy, py, vy), (fz, pz, vz) = (_stencil_1d(fine.nx + 1),
                                                _stencil_1d(fine.ny + 1),
                                                _stencil_1d(fine.nz + 1))
    ix = np.tile(np.arange(fx.size), fy.size * fz.size)
    iy = np.tile(np.repeat(np.arange(fy.size), fx.size), fz.size)
    iz = np.repeat(np.arange(fz.size), fx.size * fy.size)
    fn = node_id(fine, fx[ix], fy[iy], fz[iz])
    cnode = px[ix] + (cx + 1) * (py[iy] + (cy + 1) * pz[iz])
    w = vx[ix] * vy[iy] * vz[iz]
    rows = (3 * fn[:, None] + np.arange(3)).ravel()
    cols = (3 * cnode[:, None] + np.arange(3)).ravel()
    vals = np.repeat(w, 3)
    keep = (fine.fmap[rows] >= 0) & (coarse.fmap[cols] >= 0)
    P = sp.coo_matrix((vals[keep], (fine.fmap[rows[keep]], coarse.fmap[cols[keep]])),
                      shape=(fine.n_free, coarse.n_free))
    return canon(P), coarse


def child_patterns():
    """transfer.py:110-126: (8,24,24) child-c interpolation from coarse corners."""
    pats = np.zeros((8, 24, 24))
    for c in range(8):
        for a in range(8):
            t = (CORNERS[c] + CORNERS[a]) / 2.0
            for b in range(8):
                w = np.prod(np.where(CORNERS[b] == 1, t, 1.0 - t))
                if w != 0.0:
                    for ax in range(3):
                        pats[c, 3 * a + ax, 3 * b + ax] = w
    return pats


def galerkin_l1(fine, E, ke, coarse):
    """transfer.py:129-174: per-coarse-element sum of E_c P_c^T Ke P_c."""
    pats = child_patterns()
    tri = np.array([p.T @ ke @ p for p in pats])
    e = np.arange(fine.n_elem)
    ei, ej, ek = e % fine.nx, (e // fine.nx) % fine.ny, e // (fine.nx * fine.ny)
    code = (ei % 2) + 2 * (ej % 2) + 4 * (ek % 2)
    parent = ei // 2 + coarse.nx * (ej // 2 + coarse.ny * (ek // 2))
    acc = np.zeros((coarse.n_elem, 24, 24))
    for c in range(8):
        s = code == c
        if s.any():
            acc[parent[s]] += E[s, None, None] * tri[c]
    touch = fine.mask[fine.edofs].any(axis=1)
    for f in np.flatnonzero(touch):
        p = pats[code[f]].copy()
        p[fine.mask[fine.edofs[f]]] = 0.0
        acc[parent[f]] += E[f] * (p.T @ ke @ p - tri[code[f]])
    cd = coarse.edofs
    r = np.repeat(cd, 24, axis=1).ravel()
    c_ = np.tile(cd, (1, 24)).ravel()
    keep = (coarse.fmap[r] >= 0) & (coarse.fmap[c_] >= 0)
    K1 = sp.coo_matrix((acc.ravel()[keep], (coarse.fmap[r[keep]], coarse.fmap[c_[keep]])),
                       shape=(coarse.n_free, coarse.n_free))
    return canon(K1)


def galerkin_next(P, K):
    """transfer.py:177-181"""
    return canon(P.T @ (K @ P))


# ----------------------------------------------------------------------------
# smoothers (smoothers.py:57-152)

def band_bound(nu, alpha):
    t = (1.0 + alpha) / (1.0 - alpha)
    return float(1.0 / np.cosh(nu * np.arccosh(t)))


def cheb(apply, b, x0, dinv, lam, nu, alpha, wt):
    """smoothers.py:67-110, carried a0 = 2/sigma, first step 1/sigma."""
    b = np.asarray(b, dtype=wt)
    dinv = np.asarray(dinv, dtype=wt)
    sig = 0.5 * (lam + alpha * lam)
    dl = 0.5 * (lam - alpha * lam)
    if x0 is None:
        x = np.zeros_like(b)
        r = b
    else:
        x = np.asarray(x0, dtype=wt).copy()
        r = b - np.asarray(apply(x), dtype=wt)
    d = wt(1.0 / sig) * (dinv * r)
    x = x + d
    a = 2.0 / sig
    for _ in range(1, nu):
        r = b - np.asarray(apply(x), dtype=wt)
        c = dl * dl * a / 4.0
        a = 1.0 / (sig - c)
        d = wt(a) * (dinv * r) + wt(a * c) * d
        x = x + d
    return np.asarray(x, dtype=np.float64)


def jacobi(apply, b, x0, dinv, omega, steps, wt):
    """smoothers.py:113-131"""
    b = np.asarray(b, dtype=wt)
    dinv = np.asarray(dinv, dtype=wt)
    if x0 is None:
        x = wt(omega) * (dinv * b)
        steps -= 1
    else:
        x = np.asarray(x0, dtype=wt).copy()
    for _ in range(steps):
        x = x + wt(omega) * (dinv * (b - np.asarray(apply(x), dtype=wt)))
    return np.asarray(x, dtype=np.float64)


def power_lambda(apply, dinv, iters, seed):
    """smoothers.py:134-152 (floor 1e-6; the caller multiplies by 1.1)."""
    dinv = np.asarray(dinv, dtype=np.float64)
    v = unit_gauss(dinv.size, seed)
    lam = 0.0
    for _ in range(iters):
        w = dinv * np.asarray(apply(v), dtype=np.float64)
        lam = float(v @ w) / float(v @ v)
        s = np.linalg.norm(w)
        if s == 0.0:
            break
        v = w / s
    return max(lam, 1e-6)


# ----------------------------------------------------------------------------
# hierarchy (hierarchy.py:52-282)

POLICY = {"fp64": ("fp64",), "fp32": ("fp32", "fp64"), "bf16": ("bf16", "fp32", "fp64")}


def _tags(policy, n):
    seq = POLICY[policy]
    return [seq[min(i, len(seq) - 1)] for i in range(n)]


class Level:
    """hierarchy.py:67-120 (diag floor, f32/bf16 copies, lambda = 1.1 * power)."""

    def __init__(self, idx, K, tag, sm, seed, iters, fine=None, lam=None):
        self.idx, self.K, self.tag, self.sm, self.fine = idx, K, tag, sm, fine
        if fine is not None:
            g, E, ke = fine
            self.n = g.n_free
            d = fine_diag(g, E, ke)
        else:
            self.n = K.shape[0]
            d = K.diagonal()
            d = np.maximum(d, 1e-14 * d.mean())
            if tag != "fp64":
                self.K32 = K.astype(np.float32)
            if tag == "bf16":
                self.K16 = self.K32.copy()
                self.K16.data = bf16(self.K32.data)
        self.diag = d
        self.dinv = 1.0 / d
        self.dinv32 = self.dinv.astype(np.float32)
        self.lam = lam if lam is not None else 1.1 * power_lambda(self.mv64, self.dinv, iters, seed)
        self.P = None

    def mv64(self, x):
        if self.fine is not None:
            g, E, ke = self.fine
            return fine_apply(g, E, ke, x, "fp64")
        return self.K @ x

    def mvtag(self, x):
        if self.fine is not None:
            g, E, ke = self.fine
            wt = np.float64 if self.tag == "fp64" else np.float32
            return fine_apply(g, E, ke, np.asarray(x, wt), self.tag)
        if self.tag == "fp64":
            return self.K @ np.asarray(x, np.float64)
        if self.tag == "bf16":
            return self.K16 @ bf16(np.asarray(x, np.float32))
        return self.K32 @ np.asarray(x, np.float32)

    def smooth(self, b, x0):
        kind, deg, alpha, omega = self.sm
        wt = np.float64 if self.tag == "fp64" else np.float32
        dinv = self.dinv if self.tag == "fp64" else self.dinv32
        if kind == "chebyshev":
            return cheb(self.mvtag, b, x0, dinv, self.lam, deg, alpha, wt)
        return jacobi(self.mvtag, b, x0, dinv, omega, deg, wt)


def coarse_pcg(lev, eps, b, steps):
    """hierarchy.py:139-162"""
    dinv = 1.0 / (lev.diag + eps)
    x = np.zeros_like(b)
    r = b.copy()
    z = dinv * r
    p = z
    rz = float(r @ z)
    for _ in range(steps):
        q = lev.mv64(p) + eps * p
        pq = float(p @ q)
        if pq <= 0.0 or not np.isfinite(pq):
            break
        a = rz / pq
        x = x + a * p
        r = r - a * q
        z = dinv * r
        rzn = float(r @ z)
        if rzn <= 0.0 or not np.isfinite(rzn):
            break
        p = z + (rzn / rz) * p
        rz = rzn
    return x


class Hier:
    """hierarchy.py:181-282 (build, clamp at odd dims, V/W cycle, coarsest)."""

    def __init__(self, g, E, ke, levels=4, policy="fp32", smoother=("chebyshev", 2, 1 / 30, 0.5),
                 coarse_steps=2, cutoff=5000, pcg_steps=80, power_seed=0, lam_cache=None):
        self.policy = policy
        self.clamped = False
        ops, Ps, grids = [None], [], [g]
        cur = g
        while len(ops) < levels:
            if cur.nx % 2 or cur.ny % 2 or cur.nz % 2:
                self.clamped = True
                break
            P, coarse = transfer(cur)
            if coarse.n_free == 0:
                break
            K = galerkin_l1(g, E, ke, coarse) if len(ops) == 1 else galerkin_next(P, ops[-1])
            Ps.append(P)
            ops.append(K)
            grids.append(coarse)
            cur = coarse
        tags = _tags(policy, len(ops))
        kind, deg, alpha, omega = smoother
        self.levels = []
        for i, K in enumerate(ops):
            sm = (kind, deg, alpha, omega) if i == 0 else (kind, coarse_steps, alpha, omega)
            lam = lam_cache[i] if lam_cache is not None and i < len(lam_cache) else None
            self.levels.append(Level(i, K, tags[i], sm, power_seed + i, 20 if i == 0 else 10,
                                     fine=(g, E, ke) if i == 0 else None, lam=lam))
        for i, P in enumerate(Ps):
            self.levels[i].P = P
        self.grids = grids
        last = self.levels[-1]
        self.eps = max(float(last.diag.mean()) * 1e-8, 1e-14)
        self.pcg_steps = pcg_steps
        self.mode = "pcg80"
        if last.n <= cutoff:
            A = fine_dense(g, E, ke) if last.fine is not None else last.K.toarray()
            try:
                self.factor = sla.cho_factor(A + self.eps * np.eye(last.n), lower=True)
                self.mode = "dense_cholesky"
            except np.linalg.LinAlgError:
                pass

    def coarsest(self, r):
        if self.mode == "dense_cholesky":
            return sla.cho_solve(self.factor, r)
        return coarse_pcg(self.levels[-1], self.eps, r, self.pcg_steps)

    def cycle(self, l, r, gamma):
        if l == len(self.levels) - 1:
            return self.coarsest(r)
        lev = self.levels[l]
        x = lev.smooth(r, None)
        for _ in range(gamma):
            d = r - np.asarray(lev.mvtag(x), np.float64)
            x = x + lev.P @ self.cycle(l + 1, lev.P.T @ d, gamma)
        return lev.smooth(r, x)

    def vcycle(self, r):
        return self.cycle(0, np.asarray(r, np.float64), 1)

    def wcycle(self, r):
        return self.cycle(0, np.asarray(r, np.float64), 2)


# ----------------------------------------------------------------------------
# outer Krylov solvers (krylov.py:68-288)

def _report(apply_K, b, x, hist, kind, normb, tol, t0):
    """krylov.py:99-110: FP64 true-residual acceptance."""
    tr = float(np.linalg.norm(b - apply_K(x)) / normb)
    ok = bool(np.isfinite(tr) and tr < tol)
    return SimpleNamespace(converged=ok, iterations=len(hist), final_true_residual=tr,
                           failure_kind="none" if ok else kind, residual_history=list(hist),
                           wall_time=time.perf_counter() - t0, x=x)


def _stagnant(best):
    """krylov.py:86-97 (50-iteration window, 1%)."""
    k = len(best)
    return k > 50 and not (best[-1] <= 0.99 * best[k - 51])


def pcg(apply_K, apply_M, b, tol=1e-6, maxiter=200):
    """krylov.py:113-165"""
    t0 = time.perf_counter()
    b = np.asarray(b, dtype=np.float64)
    normb = float(np.linalg.norm(b))
    if normb == 0.0:
        return SimpleNamespace(converged=True, iterations=0, final_true_residual=0.0,
                               failure_kind="none", residual_history=[],
                               wall_time=time.perf_counter() - t0, x=np.zeros_like(b))
    hist, best = [], []
    x = np.zeros_like(b)
    r = b.copy()
    p = np.asarray(apply_M(r), dtype=np.float64)
    rz = float(r @ p)
    target, kind = tol, "cap"
    for _ in range(maxiter):
        q = np.asarray(apply_K(p), dtype=np.float64)
        pq = float(p @ q)
        if not np.isfinite(pq) or pq == 0.0:
            kind = "non_finite"
            break
        a = rz / pq
        x = x + a * p
        r = r - a * q
        rel = float(np.linalg.norm(r) / normb)
        hist.append(rel)
        best.append(min(best[-1] if best else np.inf, rel))
        if not np.isfinite(rel):
            kind = "non_finite"
            break
        if rel < target:
            if float(np.linalg.norm(b - apply_K(x)) / normb) < tol:
                kind = "none"
                break
            if _stagnant(best):
                kind = "stagnation"
                break
            target *= 0.1
        z = np.asarray(apply_M(r), dtype=np.float64)
        rzn = float(r @ z)
        if not np.isfinite(rzn):
            kind = "non_finite"
            break
        p = z + (rzn / rz) * p
        rz = rzn
    return _report(apply_K, b, x, hist, kind, normb, tol, t0)


def _upper_solve(R, g):
    """krylov.py:272-281"""
    with np.errstate(divide="ignore", invalid="ignore"):
        try:
            y = sla.solve_triangular(R, g, lower=False, check_finite=False)
        except Exception:
            y = None
    if y is None or not np.isfinite(y).all():
        y = np.linalg.lstsq(R, g.copy(), rcond=None)[0]
    return y


def fgmres(apply_K, apply_M, b, tol=1e-6, maxiter=200, restart=32):
    """krylov.py:168-269: restarted right-preconditioned flexible GMRES (MGS, Givens)."""
    t0 = time.perf_counter()
    b = np.asarray(b, dtype=np.float64)
    normb = float(np.linalg.norm(b))
    if normb == 0.0:
        return SimpleNamespace(converged=True, iterations=0, final_true_residual=0.0,
                               failure_kind="none", residual_history=[],
                               wall_time=time.perf_counter() - t0, x=np.zeros_like(b))
    hist, best = [], []
    n, m = b.size, restart
    x = np.zeros_like(b)
    kind, done = "cap", False
    while not done and len(hist) < maxiter:
        r = b - np.asarray(apply_K(x), dtype=np.float64)
        beta = float(np.linalg.norm(r))
        if not np.isfinite(beta):
            kind = "non_finite"
            break
        if beta / normb < tol:
            kind = "none"
            break
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        used, claimed = 0, False
        for j in range(m):
            Z[j] = np.asarray(apply_M(V[j]), dtype=np.float64)
            w = np.array(apply_K(Z[j]), dtype=np.float64, copy=True)
            for i in range(j + 1):
                H[i, j] = float(w @ V[i])
                w -= H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            if not np.isfinite(H[: j + 2, j]).all():
                kind, done, used = "non_finite", True, j + 1
                break
            happy = H[j + 1, j] < 1e-14
            if not happy:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j], sn[j] = (1.0, 0.0) if den == 0.0 else (H[j, j] / den, H[j + 1, j] / den)
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            used = j + 1
            rel = abs(g[j + 1]) / normb
            hist.append(float(rel))
            best.append(min(best[-1] if best else np.inf, float(rel)))
            if not np.isfinite(rel):
                kind, done = "non_finite", True
                break
            if happy or rel < tol:
                claimed = True
                break
            if len(hist) >= maxiter:
                break
        if kind == "non_finite":
            break
        if used > 0:
            x = x + Z[:used].T @ _upper_solve(H[:used, :used], g[:used])
        if done:
            break
        if float(np.linalg.norm(b - apply_K(x)) / normb) < tol:
            kind = "none"
            break
        if claimed and _stagnant(best):
            kind = "stagnation"
            break
        if len(hist) >= maxiter:
            kind = "cap"
            break
    return _report(apply_K, b, x, hist, kind, normb, tol, t0)


def jacobi_pcg(g, E, ke, b, tol=1e-6, maxiter=200):
    """krylov.py:284-288"""
    dinv = 1.0 / fine_diag(g, E, ke)
    return pcg(lambda v: fine_apply(g, E, ke, v, "fp64"), lambda r: dinv * r, b, tol, maxiter)


# ----------------------------------------------------------------------------
# spectral probe (diagnostics.py:38-92)

def lanczos_kappa(apply, n, m=40, seed=0):
    """diagnostics.py:38-79: two-pass full reorthogonalisation, eig of projected H."""
    Q = np.zeros((m, n))
    Q[0] = unit_gauss(n, seed)
    H = np.zeros((m, m))
    used, partial = m, False
    for j in range(m):
        w = np.asarray(apply(Q[j]), dtype=np.float64)
        h = Q[: j + 1] @ w
        H[: j + 1, j] = h
        w -= Q[: j + 1].T @ h
        h2 = Q[: j + 1] @ w
        H[: j + 1, j] += h2
        w -= Q[: j + 1].T @ h2
        if j == m - 1:
            break
        s = float(np.linalg.norm(w))
        if not np.isfinite(s) or s < 1e-14:
            used, partial = j + 1, True
            break
        H[j + 1, j] = s
        Q[j + 1] = w / s
    ritz = np.sort(np.linalg.eigvals(H[:used, :used]).real)
    lo, hi = float(ritz[0]), float(ritz[-1])
    kappa = hi / lo if lo != 0.0 else np.inf
    return SimpleNamespace(m=m, seed=seed, kappa_eff=float(kappa), eps_kappa=float(2.0**-8 * kappa),
                           lambda_min=lo, lambda_max=hi, partial=partial)


# ----------------------------------------------------------------------------
# convenience: the BASELINE problem set-up (bench/runner.py:37-78)

def problem(nx, ny, nz, kind="uniform", vf=0.5, p=3.0, floor=1e-2, seed=42, nu=0.3):
    g = cantilever(nx, ny, nz)
    E = simp(density(kind, nx, ny, nz, vf=vf, floor=floor, seed=seed), p)
    return g, E, element_ke(nu)


def solve(g, E, ke, policy="fp32", levels=4, method=None, tol=1e-6, maxiter=200, restart=32):
    """bench/runner.py:66-78 wiring: pcg(op.matvec, h.vcycle) or fgmres / flat Jacobi."""
    b = g.load[g.free]
    method = method or ("fgmres" if policy == "bf16" else "pcg")
    if method == "jacobi":
        return jacobi_pcg(g, E, ke, b, tol, maxiter), None
    h = Hier(g, E, ke, levels, policy)
    K = lambda v: fine_apply(g, E, ke, v, "fp64")
    if method == "pcg":
        return pcg(K, h.vcycle, b, tol, maxiter), h
    return fgmres(K, h.vcycle, b, tol, maxiter, restart), h
