"""The device dense sampled-row matvec (the north_star's sampled-row residual,
SURVEY §8d(ii); kernel entries as kernel.hpp:64-102) against the oracle's CPU
rows matvec on the same tree-order points."""
import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
import pyoracle as O
from helpers import rel, sampled_rows
from paper_1703_06155_b200.geometry import vie_constants, vie_grid_points

pytestmark = pytest.mark.gpu


def test_rows_matvec_matches_oracle():
    k0, scale, diag = vie_constants(16, 0.5)
    pts = vie_grid_points(16, 0.5)
    t = O.Tree(pts, 32)
    pts_tree = t.points
    n = pts.shape[0]
    rng = np.random.default_rng(5)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    rows = sampled_rows(n, 512, seed=7)
    yo = t.kernel_rows_matvec(O.helmholtz(k0, diag, scale), rows, x)
    yg = h2g.kernel_rows_matvec(pts_tree, h2g.helmholtz_kernel(k0, diag, scale), rows, x)
    assert rel(yg, yo) < 1e-13
    # multi-column and the residual helper
    X = np.stack([x, 2 * x], axis=1)
    Y = h2g.kernel_rows_matvec(pts_tree, h2g.helmholtz_kernel(k0, diag, scale), rows, X)
    assert rel(Y[:, 1], 2 * yo) < 1e-13
    b = np.zeros(n, np.complex128)
    b[rows] = yo
    assert h2g.sampled_dense_residual(pts_tree, h2g.helmholtz_kernel(k0, diag, scale), x, b, rows) < 1e-13


def test_rows_matvec_rejects_bad_rows():
    pts = vie_grid_points(4, 0.5)
    with pytest.raises(h2g.InvalidInputError):
        h2g.kernel_rows_matvec(pts, h2g.laplace_kernel(1.0), np.array([0, 64]), np.ones(64, np.complex128))
