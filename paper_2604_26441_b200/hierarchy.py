"""Geometric-multigrid hierarchy on the B200 (reference: hierarchy.py:1-297).

``build_hierarchy`` assembles every coarse operator on the device (level 1
by element-wise Galerkin aggregation, deeper levels by the ordered sparse
triple product), estimates lambda_max per level with device power
iterations, and sets up the coarsest solver (dense Cholesky inverse or the
persistent pcg80 kernel).  ``vcycle`` / ``wcycle`` run entirely on the GPU.
The host only supplies setup constants computed with numpy exactly as the
reference computes them (the 8 child triples P_c^T Ke P_c and the masked
Dirichlet corrections), so level 1 is bit-identical to the reference.
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _dev, _native
from .fine_operator import FineOperator
from .grid import make_grid
from .precision import PrecisionTag
from .smoothers import SmootherConfig
from .transfer import TransferPair, local_prolongation_patterns

DENSE_CHOLESKY_CUTOFF = 5000
COARSE_PCG_STEPS = 80
COARSE_SMOOTH_STEPS = 2
POWER_ITERS_FINE = 20
POWER_ITERS_COARSE = 10
LAMBDA_SAFETY = 1.1
LAMBDA_CACHE_DRIFT = 0.10

PRECISION_POLICIES = {
    "fp64": (PrecisionTag.FP64,),
    "fp32": (PrecisionTag.FP32, PrecisionTag.FP64),
    "bf16": (PrecisionTag.BF16EMU, PrecisionTag.FP32, PrecisionTag.FP64),
}
_POLICY_CODE = {"fp64": 0, "fp32": 1, "bf16": 2}
_TAG_OF_CODE = {0: PrecisionTag.FP64, 1: PrecisionTag.FP32, 2: PrecisionTag.BF16EMU}


def policy_tags(policy: str, n_levels: int):
    if policy not in PRECISION_POLICIES:
        raise ValueError(f"unknown precision policy {policy!r}")
    seq = PRECISION_POLICIES[policy]
    return [seq[min(i, len(seq) - 1)] for i in range(n_levels)]


def galerkin_tables(ke: np.ndarray, codes):
    """Host constants of the level-1 aggregation (transfer.py:140-164).

    triples[c] = P_c^T Ke P_c; for every boundary code (child << 24 | mask of
    fixed local DOFs) the correction masked - triples[child], evaluated with
    the same numpy expressions (and therefore the same bits) as the reference.
    """
    pats = local_prolongation_patterns()
    triples = np.array([p.T @ ke @ p for p in pats])
    diffs = np.zeros((len(codes), 24, 24))
    for q, code in enumerate(codes):
        child = int(code) >> 24
        fixed = np.array([(int(code) >> d) & 1 for d in range(24)], dtype=bool)
        p = pats[child].copy()
        p[fixed] = 0.0
        diffs[q] = p.T @ ke @ p - triples[child]
    return np.ascontiguousarray(triples), np.ascontiguousarray(diffs)


class _Level:
    """One hierarchy level: operator, diagonal, spectral estimate, tag."""

    _sg_native = True

    def __init__(self, h: "GmgHierarchy", index: int, info, smoother: SmootherConfig):
        self._h = h
        self.index = index
        self.tag = _TAG_OF_CODE[info.tag]
        self.smoother = smoother
        self.n_free = int(info.n_free)
        self.lam_max = float(info.lam_max)
        self.is_fine = index == 0
        self._dims = (info.nx, info.ny, info.nz)
        self._nnz = int(info.nnz)
        self._diag = None
        self._csr = None
        self._grid = None
        self.transfer: TransferPair | None = None

    # --- data views -----------------------------------------------------
    @property
    def grid(self):
        if self.is_fine:
            return self._h._op.grid
        if self._grid is None:
            nx, ny, nz = self._dims
            mask = np.zeros(3 * (nx + 1) * (ny + 1) * (nz + 1), dtype=np.uint8)
            _native.check(self._h._lib.sg_hier_level_mask(self._h._hh, self.index,
                                                          mask.ctypes.data))
            self._grid = make_grid(nx, ny, nz, mask.astype(bool))
        return self._grid

    @property
    def diag(self) -> np.ndarray:
        if self._diag is None:
            d = _dev.empty(self.n_free)
            _native.check(self._h._lib.sg_hier_level_diag(self._h._hh, self.index, _dev.ptr(d),
                                                          _dev.stream()))
            self._diag = d.cpu().numpy()
        return self._diag

    @property
    def diag_inv(self) -> np.ndarray:
        return 1.0 / self.diag

    @property
    def operator(self):
        """FineOperator on level 0, the canonical scipy CSR operator elsewhere."""
        if self.is_fine:
            return self._h._op
        if self._csr is None:
            import scipy.sparse as sp
            n = self.n_free
            indptr = np.zeros(n + 1, dtype=np.int64)
            indices = np.zeros(max(self._nnz, 1), dtype=np.int64)
            data = np.zeros(max(self._nnz, 1))
            _native.check(self._h._lib.sg_hier_level_csr(self._h._hh, self.index,
                                                         indptr.ctypes.data, indices.ctypes.data,
                                                         data.ctypes.data))
            nnz = int(indptr[-1])
            self._csr = sp.csr_matrix((data[:nnz], indices[:nnz].astype(np.int32),
                                       indptr.astype(np.int32)), shape=(n, n))
            self._csr.has_sorted_indices = True
        return self._csr

    # --- device operations ---------------------------------------------
    def _apply(self, x, tag: PrecisionTag):
        wt = tag.working_dtype
        xd, host = _dev.as_device(x, wt, self.n_free)
        y = _dev.empty(self.n_free, wt)
        _native.check(self._h._lib.sg_hier_level_apply(self._h._hh, self.index, tag.code,
                                                       _dev.ptr(xd), _dev.ptr(y), _dev.stream()))
        return _dev.back(y, host)

    def matvec64(self, x):
        return self._apply(x, PrecisionTag.FP64)

    def matvec_tagged(self, x):
        return self._apply(x, self.tag)

    def smooth(self, b, x0):
        bd, host = _dev.as_device(b, np.float64, self.n_free)
        out = _dev.empty(self.n_free)
        x0p = None
        if x0 is not None:
            x0d, _ = _dev.as_device(x0, np.float64, self.n_free)
            x0p = _dev.ptr(x0d)
        _native.check(self._h._lib.sg_hier_level_smooth(self._h._hh, self.index, _dev.ptr(bd),
                                                        x0p, _dev.ptr(out), _dev.stream()))
        return _dev.back(out, host)


@dataclass
class CoarsestSolve:
    """Regularized coarsest solver: dense Cholesky or fixed-count PCG."""

    mode: str
    eps: float
    pcg_steps: int = COARSE_PCG_STEPS
    _h: object = None

    _sg_native = True

    def solve(self, r):
        n = self._h.levels[-1].n_free
        rd, host = _dev.as_device(r, np.float64, n)
        x = _dev.empty(n)
        _native.check(self._h._lib.sg_hier_coarsest_solve(self._h._hh, _dev.ptr(rd), _dev.ptr(x),
                                                          _dev.stream()))
        return _dev.back(x, host)


class GmgHierarchy:
    """Device-resident multigrid hierarchy over one frozen modulus field."""

    _sg_native = True

    def __init__(self, op: FineOperator, hh, policy: str, max_modulus: float,
                 smoother: SmootherConfig, coarse_cfg: SmootherConfig, pcg_steps: int):
        self._op = op
        self._hh = hh
        self._lib = _native.load()
        self.policy = policy
        self.max_modulus = max_modulus
        info = _native.HierInfo()
        _native.check(self._lib.sg_hier_get_info(hh, ctypes.byref(info)))
        self.clamped = bool(info.clamped)
        self.levels = []
        for i in range(info.n_levels):
            li = _native.LevelInfo()
            _native.check(self._lib.sg_hier_level_info(hh, i, ctypes.byref(li)))
            self.levels.append(_Level(self, i, li, smoother if i == 0 else coarse_cfg))
        for i in range(info.n_levels - 1):
            self.levels[i].transfer = TransferPair._from_hierarchy(self, i)
        self.coarsest = CoarsestSolve("dense_cholesky" if info.coarsest_dense else "pcg80",
                                      float(info.eps), pcg_steps, self)

    def __del__(self):
        hh = getattr(self, "_hh", None)
        if hh is not None and hh.value:
            try:
                self._lib.sg_hier_destroy(hh)
            except Exception:
                pass
            self._hh = None

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def n_free(self) -> int:
        return self.levels[0].n_free

    def _cycle(self, r, gamma):
        n = self.n_free
        rd, host = _dev.as_device(r, np.float64, n)
        z = _dev.empty(n)
        _native.check(self._lib.sg_hier_cycle(self._hh, gamma, _dev.ptr(rd), _dev.ptr(z),
                                              _dev.stream()))
        return _dev.back(z, host)

    def vcycle(self, r):
        """One V-cycle with zero initial guess applied to a fine residual."""
        return self._cycle(r, 1)

    def wcycle(self, r):
        """One W-cycle (two coarse visits per level)."""
        return self._cycle(r, 2)


def build_hierarchy(op: FineOperator, levels: int = 4, policy: str = "fp32",
                    smoother: SmootherConfig | None = None, *,
                    coarse_smooth_steps: int = COARSE_SMOOTH_STEPS,
                    cholesky_cutoff: int = DENSE_CHOLESKY_CUTOFF,
                    coarse_pcg_steps: int = COARSE_PCG_STEPS,
                    power_seed: int = 0,
                    lambda_cache: GmgHierarchy | None = None) -> GmgHierarchy:
    """Transfers, Galerkin operators, diagonals and spectral estimates on the GPU."""
    if levels < 1:
        raise ValueError("need at least one level")
    if policy not in PRECISION_POLICIES:
        raise ValueError(f"unknown precision policy {policy!r}")
    if not isinstance(op, FineOperator):
        raise TypeError("build_hierarchy needs a paper_2604_26441_b200.FineOperator")
    smoother = smoother or SmootherConfig()
    max_E = float(np.max(op.modulus.E))
    cached = None
    if lambda_cache is not None and lambda_cache.max_modulus > 0:
        drift = abs(max_E - lambda_cache.max_modulus) / lambda_cache.max_modulus
        if drift <= LAMBDA_CACHE_DRIFT:
            cached = np.array([lev.lam_max for lev in lambda_cache.levels], dtype=np.float64)
    coarse_cfg = SmootherConfig(smoother.kind, coarse_smooth_steps, smoother.alpha, smoother.omega)
    lib = _native.load()
    # size query first (codes = NULL): user Dirichlet masks can produce any
    # number of distinct (child, local-mask) codes
    ncodes = ctypes.c_int()
    _native.check(lib.sg_fine_boundary_codes(op.handle, None, 0, ctypes.byref(ncodes)))
    cap = max(1, ncodes.value)
    codes = np.zeros(cap, dtype=np.uint32)
    _native.check(lib.sg_fine_boundary_codes(op.handle, codes.ctypes.data, cap,
                                             ctypes.byref(ncodes)))
    codes = codes[: ncodes.value]
    triples, diffs = galerkin_tables(op.ke, codes)
    p = _native.HierParams(levels, _POLICY_CODE[policy], 0 if smoother.kind == "chebyshev" else 1,
                           smoother.degree, smoother.alpha, smoother.omega, coarse_smooth_steps,
                           cholesky_cutoff, coarse_pcg_steps, power_seed)
    hh = ctypes.c_void_p()
    _native.check(lib.sg_hier_create(op.handle, ctypes.byref(p), triples.ctypes.data,
                                     codes.ctypes.data if codes.size else None,
                                     diffs.ctypes.data if codes.size else None, int(codes.size),
                                     cached.ctypes.data if cached is not None else None,
                                     0 if cached is None else int(cached.size),
                                     _dev.stream(), ctypes.byref(hh)))
    h = GmgHierarchy(op, hh, policy, max_E, smoother, coarse_cfg, coarse_pcg_steps)
    if h.clamped:
        last = h.levels[-1]
        nx, ny, nz = last._dims
        warnings.warn(f"hierarchy clamped to {h.n_levels} levels: grid ({nx},{ny},{nz}) has "
                      "an odd dimension", stacklevel=2)
    return h


def symmetry_defect(h: GmgHierarchy, n_trials: int = 10, seed: int = 0) -> float:
    """max |<Mx, y> - <x, My>| / (|x||y|) over seeded probe pairs (hierarchy.py:285-297)."""
    from . import _vec
    from .prng import SplitMix64
    if n_trials < 1:
        raise ValueError("need at least one trial")
    gen = SplitMix64(seed)
    n = h.n_free
    worst = 0.0
    for _ in range(n_trials):
        x, _ = _dev.as_device(gen.gaussian(n))
        y, _ = _dev.as_device(gen.gaussian(n))
        d = abs(_vec.dot(h.vcycle(x), y) - _vec.dot(x, h.vcycle(y)))
        worst = max(worst, d / (_vec.norm(x) * _vec.norm(y)))
    return worst
