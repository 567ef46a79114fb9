"""Explicit-inverse apply of NRHS right-hand sides on config N (waves of
right-hand-side groups): time, residual of the last column, agreement of
column 0 with the single-RHS solve.

usage: python scripts/many_rhs.py [CONFIG] [NRHS]"""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 256
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
B = np.stack([h2g.random_rhs(A.n, 1234 + j) for j in range(nrhs)], axis=1)
ms = []
for _ in range(2):
    X = ch.apply_inverse_explicit(B)
    ms.append(ch.timing()["solve_ms"])
x0 = ch.apply_inverse_explicit(B[:, 0].copy())
print("config %d: %d RHS explicit-inverse apply %.1f ms (%.2f ms per column), residual last column %.3e, column 0 vs single-RHS apply %.1e" % (
    cfg, nrhs, min(ms), min(ms) / nrhs, A.relative_residual(X[:, -1], B[:, -1]), float(np.abs(X[:, 0] - x0).max() / np.abs(x0).max())), flush=True)
