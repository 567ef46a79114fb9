"""Debug helper: per-level rank comparison of GPU vs oracle on a small case."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
sys.path.insert(0, "tests")
import paper_1703_06155_b200 as h2g  # noqa: E402
import pyoracle as O  # noqa: E402
from helpers import rod_problem, vie_problem  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "rod"
if case == "rod":
    A = rod_problem(256, 1e-12, leaf=32)
    eps = 1e-14
else:
    A, _ = vie_problem(16, 0.5, 32, 1e-4)
    eps = 1e-4
och = A.factorize(eps)
gch = h2g.factorize(h2g.H2Matrix.upload(A.arrays()), eps)
for li in range(och.num_levels):
    ro = {r["cluster"]: r for r in och.records(li)}
    rg = {r["cluster"]: r for r in gch.records(li)}
    print("level", och.level(li)["level"], "oracle diag", och.level(li), "\n        gpu diag", gch.level(li))
    for c in sorted(ro):
        a, b = ro[c], rg[c]
        if a["rank_after"] != b["rank_after"] or a["pos"] != b["pos"] or a["bsize"] != b["bsize"]:
            print("  cluster", c, "oracle", {k: a[k] for k in ("pos", "bsize", "rank_before", "rank_after")}, "gpu",
                  {k: b[k] for k in ("pos", "bsize", "rank_before", "rank_after")})
b = O.rhs(A.n, 11)
xo, xg = och.solve(b), gch.solve(b)
print("solution rel diff", np.linalg.norm(xg - xo) / np.linalg.norm(xo))
print("gpu vs shadow", np.linalg.norm(xg - A.shadow_solve(b)) / np.linalg.norm(xo) if A.n <= 4000 else "-")
