"""GPU H² construction (h2g_matrix_build, build_h2 of h2_matrix.hpp:300-375 on
the device) against the oracle's build on the same points: identical tree /
partition, ranks within +-1, compressed operator equal to construction
accuracy, and factorize+solve of the GPU-built matrix accurate against the
dense kernel."""
import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
import pyoracle as O
from helpers import rel, vie_problem
from paper_1703_06155_b200.geometry import rod_points, vie_constants, vie_grid_points

pytestmark = pytest.mark.gpu


def test_gpu_build_matches_oracle_build_vie_config1():
    eps = 1e-4
    A, K = vie_problem(16, 0.5, 32, eps)
    k0, scale, diag = vie_constants(16, 0.5)
    G = h2g.H2Matrix.build(vie_grid_points(16, 0.5), 32, 1.0, h2g.helmholtz_kernel(k0, diag, scale), eps)
    g = G.download()
    o = A.arrays()
    for k in ("cluster_begin", "cluster_end", "adm_offsets", "split_offsets"):
        assert np.array_equal(g[k], o[k]), k
    assert np.array_equal(g["perm"], A.tree.perm)
    assert np.array_equal(g["leaf_pairs"], o["leaf_pairs"])
    dr = np.abs(g["basis_rank"] - o["basis_rank"])
    assert dr.max() <= 1, dr.max()
    x = O.rhs(A.n, 5)
    # both operators approximate the kernel matrix to construction accuracy
    yo = A.matvec(x)
    yg = G.matvec(x)
    assert rel(yg, yo) < 10 * eps
    rows = np.arange(0, A.n, 7)
    yk = A.tree.kernel_rows_matvec(K, rows, x)
    assert rel(yg[rows], yk) < 10 * eps
    # oracle factorization of the GPU-built matrix (import) solves the system
    B = O.Blocks(A.tree, 1.0)
    Ag = O.H2.from_arrays(B, eps, g)
    b = O.rhs(A.n, 1234)[A.tree.perm]
    ch = h2g.factorize(G, eps)
    xg = ch.solve(b)
    assert Ag.relative_residual(xg, b) < 10 * eps
    xd = A.tree.dense_solve(K, b)
    assert rel(xg, xd) < 100 * eps


def test_gpu_build_rod_laplace():
    t = O.Tree(rod_points(400), 25)
    A = O.H2(O.Blocks(t, 1.0), O.laplace(2.0), 1e-6)
    G = h2g.H2Matrix.build(rod_points(400), 25, 1.0, h2g.laplace_kernel(2.0), 1e-6)
    x = O.rhs(400, 3)
    assert rel(G.matvec(x), A.matvec(x)) < 1e-5
    ch = h2g.factorize(G, 1e-8)
    b = O.rhs(400, 4)
    assert rel(ch.solve(b), t.dense_solve(O.laplace(2.0), b)) < 1e-4
