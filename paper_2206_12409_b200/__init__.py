"""B200-native Z_bc coupling library (hybrid VSIE, arXiv 2206.12409).

The compute path is the sm_100a C-ABI library ``libvsie_coupling.so``
(include/vsie_coupling.h); this package is its thin Python binding.
"""
from ._lib import VsieError, lib  # noqa: F401
from .coupling import Coupling, Grid, PWLCoupling, nccl_unique_id, slab_partition, set_allocator, use_torch_allocator  # noqa: F401
from .farnear import FarFar, FarNear  # noqa: F401
from .hybrid import Hybrid  # noqa: F401


def grid_of(cfg) -> Grid:
    """Grid descriptor of a synth.Config (input marshalling only)."""
    return Grid(tuple(cfg.n), tuple(cfg.h), tuple(cfg.origin))
