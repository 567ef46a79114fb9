"""Step-0 refinement switch (H2G_REFINE_BELOW) at eps below 1e-4: per-cluster
ranks, solution and time of the Gram-only truncation and of the refined one
against the CPU oracle (config 1 geometry), then both on the config-2 geometry
(no oracle at that size: residuals).

usage: python scripts/refine_switch.py [EPS]"""
import os
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
sys.path.insert(0, "tests")
import numpy as np

import paper_1703_06155_b200 as h2g
import pyoracle as O
from helpers import ranks_by_cluster, rel, vie_problem
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-6
c = BASELINE_CONFIGS[1]
t0 = time.time()
A, K = vie_problem(c["cells"], c["side"], c["leaf"], eps)
och = A.factorize(eps)
print("config-1 geometry, eps %.0e: oracle build + factorize %.1f s" % (eps, time.time() - t0), flush=True)
ro = ranks_by_cluster(och.all_records())
b = O.rhs(A.n, 1234)[A.tree.perm]
xo = och.solve(b)
G = h2g.H2Matrix.upload(A.arrays())
for below in ("1e-4", "3e-7", "1e-7"):
    os.environ["H2G_REFINE_BELOW"] = below
    for _ in range(2):
        gch = h2g.factorize(G, eps)
    rg = ranks_by_cluster(gch.all_records())
    d = np.array([rg[k] - ro[k] for k in ro])
    xg = gch.solve(b)
    print("  refine below %s sigma_0: factor %.1f ms; rank diffs vs oracle: max |d| %d, nonzero %d of %d, sum %d; x rel diff %.3e; residual oracle %.3e gpu %.3e" % (
        below, gch.timing()["factor_ms"], np.abs(d).max(), np.count_nonzero(d), len(d), d.sum(), rel(xg, xo), A.relative_residual(xo, b), A.relative_residual(xg, b)), flush=True)

c = BASELINE_CONFIGS[2]
k0, scale, diag = vie_constants(c["cells"], c["side"])
K = h2g.helmholtz_kernel(k0, diag, scale)
pts = vie_grid_points(c["cells"], c["side"])
A2 = h2g.H2Matrix.build(pts, c["leaf"], 1.0, K, eps)
perm = A2.perm()
b2 = h2g.random_rhs(A2.n, 1234)[perm]
rows = np.sort(np.random.default_rng(1234).choice(A2.n, size=4096, replace=False)).astype(np.int64)
ranks = {}
for below in ("1e-7", "3e-7") + (("1e-4",) if len(sys.argv) > 2 else ()):
    os.environ["H2G_REFINE_BELOW"] = below
    ch = h2g.factorize(A2, eps)
    x = ch.solve(b2)
    ranks[below] = ranks_by_cluster(ch.all_records())
    print("config-2 geometry, eps %.0e, refine below %s: factor %.1f ms, levels %s root %d; residual H2 %.3e, sampled dense rows %.3e" % (
        eps, below, ch.timing()["factor_ms"], [l["rank_sum_after"] for l in ch.levels()], ch.root_size, A2.relative_residual(x, b2),
        h2g.sampled_dense_residual(pts[perm], K, x, b2, rows)), flush=True)
    del ch
