"""The five BASELINE.json configurations as concrete synthetic geometry.

Paper context: the body sits in a uniform voxel box n1 x n2 x n3 (PAPER.md
P:90); the far-domain conductors are an RF shield and a scanner bore,
both open cylinders.  The paper's phantoms and coil
meshes are not available, so BASELINE.json's box grids and synthetic cylinders
stand in (SURVEY.md §8d "Datasets").

Readings adopted:
* voxel centres at (i - (n-1)/2) * h per axis, i1 <-> x, i2 <-> y, i3 <-> z;
* open cylinder about z, z in [-L/2, L/2], phi_j = 2 pi j / N_az,
  z_k = -L/2 + k L / N_ax, vertex id k*N_az + j, quad (j, k) split into
  (v_jk, v_j+1,k, v_j+1,k+1) and (v_jk, v_j+1,k+1, v_j,k+1), triangle ids
  2(k N_az + j) + {0, 1}, azimuthal seam periodic;
* f = 298.2 MHz (7 T), c0 = 299 792 458 m/s.

Everything here is an *input*: vertex coordinates and integer topology.  The
method's arithmetic (RWG extraction, quadrature, Green's function) lives in
``oracle/`` and in the CUDA library, separately.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

C0 = 299_792_458.0
FREQ_7T = 298.2e6


@dataclass(frozen=True)
class Surface:
    name: str
    radius: float
    length: float
    n_az: int
    n_ax: int

    @property
    def n_rwg(self) -> int:  # closed form, SURVEY §8c-P11
        return self.n_az * (3 * self.n_ax - 1)

    @property
    def n_tri(self) -> int:
        return 2 * self.n_az * self.n_ax


@dataclass(frozen=True)
class Config:
    idx: int
    name: str
    n: tuple
    h: tuple
    surfaces: tuple
    tol: float
    repeats: int
    nrhs: int = 1
    freq: float = FREQ_7T
    ranks_probe: tuple = field(default=())

    @property
    def origin(self) -> tuple:
        return tuple(-(self.n[a] - 1) * self.h[a] / 2.0 for a in range(3))

    @property
    def n_v(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def m(self) -> int:
        return sum(s.n_rwg for s in self.surfaces)

    @property
    def k0(self) -> float:
        return 2.0 * math.pi * self.freq / C0

    def meshes(self):
        """List of (xyz float64 [nv,3], tri int32 [nt,3]) in surface order."""
        return [cylinder_mesh(s.radius, s.length, s.n_az, s.n_ax) for s in self.surfaces]


def cylinder_mesh(radius: float, length: float, n_az: int, n_ax: int):
    """Structured open-cylinder triangle mesh."""
    j = np.arange(n_az)
    k = np.arange(n_ax + 1)
    phi = 2.0 * np.pi * j / n_az
    z = -length / 2.0 + k * length / n_ax
    xyz = np.empty(((n_ax + 1) * n_az, 3), dtype=np.float64)
    kk, jj = np.meshgrid(k, j, indexing="ij")
    vid = kk * n_az + jj
    xyz[vid.ravel(), 0] = radius * np.cos(phi[jj.ravel()])
    xyz[vid.ravel(), 1] = radius * np.sin(phi[jj.ravel()])
    xyz[vid.ravel(), 2] = z[kk.ravel()]
    tri = np.empty((2 * n_az * n_ax, 3), dtype=np.int32)
    for kq in range(n_ax):
        for jq in range(n_az):
            j1 = (jq + 1) % n_az
            v00 = kq * n_az + jq
            v10 = kq * n_az + j1
            v11 = (kq + 1) * n_az + j1
            v01 = (kq + 1) * n_az + jq
            t = 2 * (kq * n_az + jq)
            tri[t] = (v00, v10, v11)
            tri[t + 1] = (v00, v11, v01)
    return xyz, tri


_SHIELD = dict(radius=0.34, length=1.2)
_BORE = dict(radius=0.40, length=2.0)

CONFIGS = {
    1: Config(1, "tiny", (12, 12, 12), (5e-3,) * 3,
              (Surface("shield", n_az=24, n_ax=16, **_SHIELD),), tol=1e-8, repeats=50,
              ranks_probe=(7, 31, 73)),
    2: Config(2, "head2mm", (100, 120, 110), (2e-3,) * 3,
              (Surface("shield", n_az=72, n_ax=47, **_SHIELD),), tol=1e-6, repeats=50,
              ranks_probe=(10, 67, 240)),
    3: Config(3, "body2mm", (200, 120, 400), (2e-3,) * 3,
              (Surface("shield", n_az=88, n_ax=57, **_SHIELD),
               Surface("bore", n_az=80, n_ax=63, **_BORE)), tol=1e-6, repeats=50,
              ranks_probe=(16, 124, 1100)),
    4: Config(4, "head1mm", (200, 240, 220), (1e-3,) * 3,
              (Surface("shield", n_az=100, n_ax=67, **_SHIELD),
               Surface("bore", n_az=90, n_ax=74, **_BORE)), tol=1e-6, repeats=100,
              ranks_probe=(10, 63, 225)),
    5: Config(5, "block64", (200, 120, 400), (2e-3,) * 3,
              (Surface("shield", n_az=88, n_ax=57, **_SHIELD),
               Surface("bore", n_az=80, n_ax=63, **_BORE)), tol=1e-6, repeats=20, nrhs=64,
              ranks_probe=(16, 124, 1100)),
}


def get_config(i: int) -> Config:
    return CONFIGS[int(i)]


# Near-domain conductor of the 3 x 3 hybrid system ("the receive array is usually in the
# near domain"; Fig. 1): no coil meshes are available, so an open cylinder coaxial
# with the far surfaces, just outside the voxel box, stands in for the receive-array former
# (reading R-CC3).  #RWG = n_az (3 n_ax - 1).
NEAR_COILS = {
    1: Surface("near", radius=0.15, length=0.20, n_az=16, n_ax=8),     # 368 RWG
    2: Surface("near", radius=0.17, length=0.26, n_az=48, n_ax=30),    # 4272 RWG
    3: Surface("near", radius=0.26, length=0.60, n_az=64, n_ax=40),    # 7616 RWG
    4: Surface("near", radius=0.17, length=0.26, n_az=64, n_ax=40),    # 7616 RWG
    5: Surface("near", radius=0.26, length=0.60, n_az=64, n_ax=40),
}


def near_coil(i: int) -> Surface:
    return NEAR_COILS[int(i)]


def near_mesh(i: int):
    """(xyz, tri) of the near conductor of config i."""
    s = near_coil(i)
    return cylinder_mesh(s.radius, s.length, s.n_az, s.n_ax)
