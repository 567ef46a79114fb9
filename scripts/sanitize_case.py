"""Small case for compute-sanitizer (racecheck / synccheck): BASELINE config 1
geometry at eps 1e-6 (levels with blocks above 64 rows exercise the
thread-block-cluster kernels k_eig1c / k_eig1b_cl and the extended LU), the
dataflow and the batch-synchronous solves, the device residual."""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import vie_constants, vie_grid_points

k0, scale, diag = vie_constants(16, 0.5)
pts = vie_grid_points(16, 0.5)
K = h2g.helmholtz_kernel(k0, diag, scale)
A = h2g.H2Matrix.build(pts, 32, 1.0, K, 1e-6)
ch = h2g.factorize(A, 1e-6)
b = h2g.random_rhs(A.n, 1234)
x = ch.solve(b)
X = ch.apply_inverse_explicit(np.stack([b, 2 * b], axis=1))
perm = A.perm()
rows = np.arange(0, A.n, 37, dtype=np.int64)
r = h2g.sampled_dense_residual(pts[perm], K, x, b, rows)
print("levels", [(l["level"], l["rank_sum_after"]) for l in ch.levels()], "root", ch.root_size, "residual", A.relative_residual(x, b), "dense rows", r)
# the large-configuration storage paths and the SUBTREE order on the same input
os.environ["H2G_FILL_SEGMENTS"] = "4"
os.environ["H2G_CHAIN_STREAM"] = "1"
os.environ["H2G_EIG_GLOBAL"] = "1"
A.ctx.clear_plans()
A2 = h2g.H2Matrix.build(pts, 32, 1.0, K, 1e-6)
ch2 = h2g.factorize(A2, 1e-6)
x2 = ch2.solve(b)
for k in ("H2G_FILL_SEGMENTS", "H2G_CHAIN_STREAM", "H2G_EIG_GLOBAL"):
    del os.environ[k]
ch3 = h2g.factorize(A2, 1e-6, schedule="subtree")
x3 = ch3.solve(b)
print("segmented + streamed residual", A.relative_residual(x2, b), "subtree residual", A.relative_residual(x3, b))
