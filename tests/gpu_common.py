"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
import numpy as np

import synth


def rand_cores(dims, ranks, seed, scale=1.0):
    """Random complex TT cores (r_{k-1}, n_k, r_k), entries ~ N(0,1)/sqrt(r_{k-1}) (seeded)."""
    rng = np.random.default_rng(seed)
    rr = (1,) + tuple(ranks) + (1,)
    out = []
    for k in range(4):
        shp = (rr[k], dims[k], rr[k + 1])
        a = (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / np.sqrt(2 * rr[k])
        out.append(a * scale)
    return out


def rand_tts(cfg, ranks_per_chi, seed):
    dims = tuple(cfg.n) + (cfg.m,)
    return [rand_cores(dims, ranks_per_chi[c], seed + 101 * c) for c in range(3)]


def grid_of(cfg):
    from paper_2206_12409_b200 import Grid
    return Grid(tuple(cfg.n), tuple(cfg.h), tuple(cfg.origin))


def inflate(cores, extra, seed):
    """Same tensor with each inner rank grown by `extra` redundant directions:
    G_k <- [G_k, G_k M_k] on the right, G_{k+1} <- [G_{k+1}; 0] on the left."""
    rng = np.random.default_rng(seed)
    G = [np.array(c, dtype=np.complex128) for c in cores]
    for k in range(len(G) - 1):
        a, n, b = G[k].shape
        M = rng.normal(size=(b, extra)) + 1j * rng.normal(size=(b, extra))
        L = G[k].reshape((a * n, b), order="F")
        G[k] = np.concatenate([L, L @ M], axis=1).reshape((a, n, b + extra), order="F")
        b2, n2, c2 = G[k + 1].shape
        G[k + 1] = np.concatenate([G[k + 1], np.zeros((extra, n2, c2), complex)], axis=0)
    return G
