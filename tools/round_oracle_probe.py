"""Probe: time the oracle's TT rounding steps on the config-2 cross cores (diagnostics)."""
import faulthandler
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import synth  # noqa: E402
from oracle import ttround  # noqa: E402
from paper_2206_12409_b200 import Coupling, grid_of  # noqa: E402

faulthandler.dump_traceback_later(45, repeat=True)
cfg = synth.get_config(2)
h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
src = h.export_cores()[2]
print("shapes", [c.shape for c in src], "finite", [bool(np.isfinite(c).all()) for c in src], flush=True)
G = [np.array(c) for c in src]
for k in range(3, 0, -1):
    a, n, b = G[k].shape
    X = G[k].reshape((a, n * b), order="F").T
    t = time.perf_counter()
    Q, R = np.linalg.qr(X)
    print("qr", k, X.shape, time.perf_counter() - t, flush=True)
    G[k] = Q.T.reshape((Q.shape[1], n, b), order="F")
    p, m, _ = G[k - 1].shape
    G[k - 1] = (G[k - 1].reshape((p * m, a), order="F") @ R.T).reshape((p, m, Q.shape[1]), order="F")
for k in range(3):
    a, n, b = G[k].shape
    M = G[k].reshape((a * n, b), order="F")
    t = time.perf_counter()
    U, S, Vh = np.linalg.svd(M, full_matrices=False)
    print("svd", k, M.shape, time.perf_counter() - t, S[:3], flush=True)
    G[k + 1] = ((S[:, None] * Vh) @ G[k + 1].reshape((b, -1), order="F")).reshape((len(S),) + G[k + 1].shape[1:], order="F")
    G[k] = U.reshape((a, n, len(S)), order="F")
print("done", flush=True)
