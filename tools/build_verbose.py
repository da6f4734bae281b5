import sys; sys.path.insert(0, ".")
import synth
from paper_2206_12409_b200 import Coupling, grid_of
cfg = synth.get_config(int(sys.argv[1]))
h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, verbose=1)
print(h.info()["ranks"], h.info()["build_s"])
