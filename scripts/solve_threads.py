"""64-RHS explicit-inverse apply on config N for the shared-memory budgets in
argv[2:] under the H2G_SOLVE_THREADS of the environment (read once per process).

usage: H2G_SOLVE_THREADS=512 python scripts/solve_threads.py 2 150 100 64"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

cfg = int(sys.argv[1])
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
B = np.stack([h2g.random_rhs(A.n, 1234 + j) for j in range(64)], axis=1)
for kb in sys.argv[2:]:
    os.environ["H2G_SOLVE_SMEM_KB"] = kb
    ms = []
    for _ in range(3):
        X = ch.apply_inverse_explicit(B)
        ms.append(ch.timing()["solve_ms"])
    print("threads %s smem %s KB: 64-RHS apply %.1f ms, residual col 63 %.3e" % (os.environ.get("H2G_SOLVE_THREADS", "auto"), kb, min(ms), A.relative_residual(X[:, 63], B[:, 63])), flush=True)
del os.environ["H2G_SOLVE_SMEM_KB"]
b = B[:, 0].copy()
ms = []
for _ in range(6):
    x = ch.solve(b)
    ms.append(ch.timing()["solve_ms"])
print("threads %s: nrhs = 1 solve %.2f ms" % (os.environ.get("H2G_SOLVE_THREADS", "auto"), float(np.median(ms[1:]))), flush=True)
