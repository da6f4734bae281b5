"""TT-cross build with progress lines: python tools/build_verbose.py CONFIG [VERBOSE].

VERBOSE 1 prints one line per sweep and chi (ranks, held-out error, time breakdown),
2 adds one line per Jacobi call (p, q, sweeps)."""
import sys
sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2206_12409_b200 import Coupling, grid_of  # noqa: E402

cfg = synth.get_config(int(sys.argv[1]))
h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1,
                   verbose=int(sys.argv[2]) if len(sys.argv) > 2 else 1)
i = h.info()
print("build_s", i["build_s"], "factor", i["build_factor_s"], "ranks", i["ranks"], "heldout", i["heldout_err"],
      flush=True)
