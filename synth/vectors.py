"""Seeded random inputs (SURVEY.md §8c-L20, §8d "Vectors").

complex Gaussian = (a + i b)/sqrt(2), a, b iid N(0, 1), drawn by
numpy.random.Generator(PCG64(seed)).standard_normal((n, 2)).
"""
from __future__ import annotations

import numpy as np

SEEDS = dict(x=12409001, u=12409002, X=12409003, U=12409004, heldout=12409005, cross=12409010)


def complex_gaussian(n: int, seed: int, ncols: int | None = None) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    shape = (n if ncols is None else n * ncols, 2)
    a = rng.standard_normal(shape)
    z = (a[:, 0] + 1j * a[:, 1]) / np.sqrt(2.0)
    if ncols is None:
        return z
    return z.reshape((n, ncols), order="F")


def uniform_indices(dims, count: int, seed: int) -> np.ndarray:
    """count x len(dims) int64 array of uniform multi-indices."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cols = [rng.integers(0, d, size=count, dtype=np.int64) for d in dims]
    return np.stack(cols, axis=1)


def phantom_eps(n, h, origin, freq: float, eps_tissue: float = 52.0, sigma: float = 0.55) -> np.ndarray:
    """Synthetic body phantom (the paper's head / body models are not available): complex
    relative permittivity per voxel, i1 fastest (v = i1 + n1 (i2 + n2 i3)).  An ellipsoid
    filling 80% of the box along each axis holds tissue eps_r - i sigma / (omega eps0)
    (exp(+i omega t), matching g = exp(-i k0 R) / (4 pi R)); outside it is air (eps_r = 1).
    Defaults: muscle-like 52, 0.55 S/m (the 7 T range of the paper's tissue values)."""
    eps0 = 8.8541878128e-12
    c = [origin[a] + (n[a] - 1) * h[a] / 2.0 for a in range(3)]
    ax = [0.4 * n[a] * h[a] for a in range(3)]
    i1, i2, i3 = np.meshgrid(np.arange(n[0]), np.arange(n[1]), np.arange(n[2]), indexing="ij")
    r2 = sum(((origin[a] + idx * h[a] - c[a]) / ax[a]) ** 2 for a, idx in enumerate((i1, i2, i3)))
    inside = (r2 <= 1.0).transpose(2, 1, 0).reshape(-1)   # i1 fastest
    eps = np.ones(n[0] * n[1] * n[2], dtype=np.complex128)
    eps[inside] = eps_tissue - 1j * sigma / (2 * np.pi * freq * eps0)
    return eps
