"""Factorize config N once, then time the solve (nrhs 1 and 64) and print
the residuals (used to compare the dataflow and batch-synchronous kernels)."""
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
b = h2g.random_rhs(A.n, 1234)
ms = []
for _ in range(6):
    x = ch.solve(b)
    ms.append(ch.timing()["solve_ms"])
B = np.stack([h2g.random_rhs(A.n, 1234 + j) for j in range(64)], axis=1)
X = ch.apply_inverse_explicit(B)
ms64 = ch.timing()["solve_ms"]
print("solve ms nrhs=1 %.2f (median of 5 after warm-up), nrhs=64 %.1f; residual %.3e, col 63 %.3e, x[0:2] %s" % (
    float(np.median(ms[1:])), ms64, A.relative_residual(x, b), A.relative_residual(X[:, 63], B[:, 63]), x[:2]))
