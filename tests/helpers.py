"""Shared fixtures: identical seeded inputs for the oracle and the GPU path."""
import numpy as np

import pyoracle as O
from paper_1703_06155_b200.geometry import rod_points, vie_constants, vie_grid_points


def rod_problem(n, eps_h2, leaf=25, eta=1.0, kernel=None):
    kernel = kernel or O.laplace(2.0)
    t = O.Tree(rod_points(n), leaf)
    b = O.Blocks(t, eta)
    return O.H2(b, kernel, eps_h2)


def vie_problem(cells, side, leaf, eps):
    k0, scale, diag = vie_constants(cells, side)
    K = O.helmholtz(k0, diag, scale)
    t = O.Tree(vie_grid_points(cells, side), leaf)
    b = O.Blocks(t, 1.0)
    return O.H2(b, K, eps), K


def ranks_by_cluster(records):
    return {(r["level"], r["cluster"]): r["rank_after"] for r in records}


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
