"""Factorize config N once, then time the 64-RHS explicit-inverse apply with
the right-hand-side groups side by side (one launch per level, grid y) and one
after the other, for several shared-memory budgets per CTA.

usage: python scripts/solve_groups.py [CONFIG] [EPS]"""
import os
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = dict(BASELINE_CONFIGS[cfg])
if len(sys.argv) > 2:
    c["eps"] = float(sys.argv[2])
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
print("config %d eps %.0e factorized: %s" % (cfg, c["eps"], ch.timing()), flush=True)
B = np.stack([h2g.random_rhs(A.n, 1234 + j) for j in range(64)], axis=1)
ref = None
for kb in (150, 100, 64, 40):
    for groups in (0, 1):
        os.environ["H2G_SOLVE_SMEM_KB"] = str(kb)
        os.environ["H2G_SOLVE_GROUPS"] = str(groups)
        ms = []
        for _ in range(3):
            X = ch.apply_inverse_explicit(B)
            ms.append(ch.timing()["solve_ms"])
        if ref is None:
            ref = X
        print("smem %3d KB, groups %s: 64-RHS apply %.1f ms (best of 3: %s), max |X - X_first| / |X| %.1e, residual col 63 %.3e" % (
            kb, "side by side" if groups else "sequential", min(ms), ["%.1f" % m for m in ms],
            float(np.abs(X - ref).max() / np.abs(ref).max()), A.relative_residual(X[:, 63], B[:, 63])), flush=True)
del os.environ["H2G_SOLVE_SMEM_KB"], os.environ["H2G_SOLVE_GROUPS"]
b = B[:, 0].copy()
ms = []
for _ in range(6):
    x = ch.solve(b)
    ms.append(ch.timing()["solve_ms"])
print("nrhs = 1 solve %.2f ms (median of 5)" % float(np.median(ms[1:])))
