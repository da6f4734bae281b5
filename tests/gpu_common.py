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
