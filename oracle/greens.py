"""Oracle — free-space Green's function and its dyad (Eq. 3).

  G(r, r') = (I + grad grad / k0^2) g(r, r'),   g = exp(-i k0 R) / (4 pi R)

Reading §8c-L2: the printed extra 1/(4 pi) in front of the dyad is
dropped (g already carries 1/(4 pi R)); scalar-only.  §8c-L3: the phase sign
exp(-i k0 R) is kept as printed.

Closed form of the dyad (derived by differentiating g twice):
  G(R) = g(R) [ alpha I + beta Rhat Rhat^T ],
  alpha = 1 - i u - u^2,  beta = -1 + 3 i u + 3 u^2,  u = 1/(k0 R).
Pinned in tests against 40-digit mpmath finite differences of g (P2), the
Helmholtz trace identity tr G = 2 g (P1) and symmetry (P3).
"""
from __future__ import annotations

import numpy as np


def g_scalar(R, k0):
    """g = exp(-i k0 R)/(4 pi R)."""
    R = np.asarray(R, dtype=np.float64)
    return np.exp(-1j * k0 * R) / (4.0 * np.pi * R)


def dyad(Rvec, k0):
    """Full 3x3 dyad G(R) for R = r - r' (shape [..., 3] -> [..., 3, 3])."""
    Rvec = np.asarray(Rvec, dtype=np.float64)
    R = np.asarray(np.linalg.norm(Rvec, axis=-1))
    rh = Rvec / R[..., None]
    u = 1.0 / (k0 * R)
    alpha = np.asarray(1.0 - 1j * u - u * u)
    beta = np.asarray(-1.0 + 3j * u + 3.0 * u * u)
    g = np.asarray(g_scalar(R, k0))
    eye = np.eye(3)
    return g[..., None, None] * (alpha[..., None, None] * eye
                                 + beta[..., None, None] * rh[..., :, None] * rh[..., None, :])


def dyad_apply(Rvec, J, k0):
    """G(R) J for real vectors J (shape [..., 3]) without forming the 3x3."""
    Rvec = np.asarray(Rvec, dtype=np.float64)
    R = np.asarray(np.sqrt(np.sum(Rvec * Rvec, axis=-1)))
    rh = Rvec / R[..., None]
    u = 1.0 / (k0 * R)
    alpha = np.asarray(1.0 - 1j * u - u * u)
    beta = np.asarray(-1.0 + 3j * u + 3.0 * u * u)
    g = np.asarray(g_scalar(R, k0))
    rj = np.sum(rh * J, axis=-1)
    return g[..., None] * (alpha[..., None] * J + (beta * rj)[..., None] * rh)
