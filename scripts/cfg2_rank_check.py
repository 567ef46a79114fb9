"""Per-level rank deviation of the GPU factorization of config 2 from the
committed oracle fixture, next to the oracle's own rank noise
(tests/golden/cfg2_rank_noise.json); run with H2G_DEBUG=4 to force the step-0
refinement pass at every cluster."""
import json
import os
import sys
import time

sys.path[:0] = [".", "tests"]
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

G = "tests/golden"
gold = np.load(os.path.join(G, "cfg2_oracle.npz"))
noise = json.load(open(os.path.join(G, "cfg2_rank_noise.json")))
c = BASELINE_CONFIGS[2]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
for rep in range(2):
    t0 = time.time()
    ch = h2g.factorize(A, c["eps"])
    wall = time.time() - t0
ro = {(int(r[0]), int(r[1])): int(r[4]) for r in gold["rec"]}
rg = {(r["level"], r["cluster"]): r["rank_after"] for r in ch.all_records()}
print("H2G_DEBUG", os.environ.get("H2G_DEBUG"), "factor_ms %.1f wall %.2f s" % (ch.timing()["factor_ms"], wall))
for lv in sorted({k[0] for k in ro}, reverse=True):
    d = np.array([rg[k] - ro[k] for k in ro if k[0] == lv])
    print("level %d: gpu max|d| %d mean %.2f sum %d vs oracle %d | oracle noise max %d mean %.2f" % (
        lv, np.abs(d).max(), np.abs(d).mean(), sum(v for k, v in rg.items() if k[0] == lv), sum(v for k, v in ro.items() if k[0] == lv),
        noise["per_level"][str(lv)]["max_abs"], noise["mean_abs_per_level"][str(lv)]))
