"""Point clouds and the BASELINE VIE problem definition (host side).

Geometry generators follow proj/include/h2lu/geometry.hpp:54-82 (rod, slab,
cube). The volume-integral-equation (Lippmann-Schwinger) cube of BASELINE.json
follows SURVEY.md §8d: lambda = 1, k0 = 2 pi, eps_r = 4, cell-centred grid
with x fastest (original index p = ix + n*iy + n^2*iz).
"""
from __future__ import annotations

import math

import numpy as np


def rod_points(n, spacing=1.0):
    pts = np.zeros((n, 3))
    pts[:, 0] = np.arange(n, dtype=np.float64) * spacing
    return pts


def slab_points(n, spacing=1.0):
    side = int(math.ceil(math.sqrt(float(n))))
    i = np.arange(n)
    pts = np.zeros((n, 3))
    pts[:, 0] = (i % side) * spacing
    pts[:, 1] = (i // side) * spacing
    return pts


def cube_points(n, spacing=1.0):
    side = int(math.ceil(np.cbrt(float(n))))
    while side ** 3 < n:
        side += 1
    i = np.arange(n)
    pts = np.zeros((n, 3))
    pts[:, 0] = (i % side) * spacing
    pts[:, 1] = ((i // side) % side) * spacing
    pts[:, 2] = (i // (side * side)) * spacing
    return pts


def vie_grid_points(cells_per_side, side_lambda):
    """Cell centres of an n^3 grid over a cube of side `side_lambda` (lambda = 1)."""
    n = cells_per_side
    h = side_lambda / n
    p = np.arange(n ** 3)
    ix, iy, iz = p % n, (p // n) % n, p // (n * n)
    return np.stack([(ix + 0.5) * h, (iy + 0.5) * h, (iz + 0.5) * h], axis=1)


def vie_constants(cells_per_side, side_lambda, eps_r=4.0):
    """(k0, off-diagonal scale, complex self term) of the BASELINE VIE.

    A_ij = k0^2 (eps_r - 1) h^3 exp(-j k0 r)/(4 pi r) for i != j and
    A_ii = 1 + 2 (eps_r - 1) [(1 + j k0 a) exp(-j k0 a) - 1], a = (3/(4 pi))^(1/3) h.
    """
    h = side_lambda / cells_per_side
    k0 = 2.0 * math.pi
    scale = k0 * k0 * (eps_r - 1.0) * h ** 3
    a = (3.0 / (4.0 * math.pi)) ** (1.0 / 3.0) * h
    diag = 1.0 + 2.0 * (eps_r - 1.0) * ((1.0 + 1j * k0 * a) * np.exp(-1j * k0 * a) - 1.0)
    return k0, scale, complex(diag)


# BASELINE.json configs: (cells per side, cube side in wavelengths, leaf size, eps)
BASELINE_CONFIGS = {
    1: dict(cells=16, side=0.5, leaf=32, eps=1e-4),
    2: dict(cells=32, side=1.0, leaf=32, eps=1e-4),
    3: dict(cells=64, side=4.0, leaf=64, eps=1e-4),
    4: dict(cells=64, side=4.0, leaf=64, eps=1e-4),
    5: dict(cells=128, side=8.0, leaf=64, eps=1e-3),
}
