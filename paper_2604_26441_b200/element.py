"""Unit-modulus Q1 hexahedral element stiffness (reference: element.py:1-70).

24x24, 2x2x2 Gauss quadrature on the unit cube, isotropic material with
Poisson ratio nu.  Host constant: computed with the same numpy expression
order as the reference so its bits (and every bit-exact Galerkin product
built from it) match on the same host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import CORNER_OFFSETS


@dataclass(frozen=True)
class ElementStiffness:
    ke: np.ndarray
    nu: float


def _constitutive(nu):
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2.0 * mu
    D[3:, 3:] = mu * np.eye(3)
    return D


def _strain_matrix(dn):
    """6x24 small-strain operator from shape-function gradients dn (8, 3)."""
    B = np.zeros((6, 24))
    for a in range(8):
        gx, gy, gz = dn[a]
        c = 3 * a
        B[0, c] = gx
        B[1, c + 1] = gy
        B[2, c + 2] = gz
        B[3, c], B[3, c + 1] = gy, gx
        B[4, c + 1], B[4, c + 2] = gz, gy
        B[5, c], B[5, c + 2] = gz, gx
    return B


def unit_element_stiffness(nu: float = 0.3) -> ElementStiffness:
    if not (0.0 <= nu < 0.5):
        raise ValueError(f"Poisson ratio must lie in [0, 0.5), got {nu}")
    D = _constitutive(nu)
    sign = 2.0 * CORNER_OFFSETS - 1.0
    g = 1.0 / np.sqrt(3.0)
    ke = np.zeros((24, 24))
    for p in (-g, g):
        for q in (-g, g):
            for r in (-g, g):
                f = 1.0 + sign * np.array([p, q, r])
                dn = np.empty((8, 3))
                dn[:, 0] = sign[:, 0] * f[:, 1] * f[:, 2]
                dn[:, 1] = f[:, 0] * sign[:, 1] * f[:, 2]
                dn[:, 2] = f[:, 0] * f[:, 1] * sign[:, 2]
                dn *= 2.0 / 8.0
                B = _strain_matrix(dn)
                ke += (B.T @ D @ B) / 8.0
    ke = 0.5 * (ke + ke.T)
    ke.setflags(write=False)
    return ElementStiffness(ke, nu)
