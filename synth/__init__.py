"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no Green's function, no RWG
extraction, no quadrature, no TT algebra).  It only produces *inputs*:

* voxel-grid descriptors (n, h, origin) for the BASELINE.json configs,
* open-cylinder triangle meshes (vertex xyz + triangle vertex ids) that stand in
  for the RF shield and the scanner bore,
* seeded complex Gaussian vectors and uniform index samples (§8c-L20, §8d).

Both ``oracle/`` and ``paper_2206_12409_b200`` may import it; it imports
neither.
"""
from .configs import CONFIGS, Config, Surface, cylinder_mesh, get_config, near_coil, near_mesh  # noqa: F401
from .vectors import complex_gaussian, phantom_eps, uniform_indices, SEEDS  # noqa: F401
