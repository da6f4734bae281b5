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
