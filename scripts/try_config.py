"""Build and factorize one BASELINE config with level logging; report ranks, time, residual."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
t0 = time.time()
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
print("build %.1f s" % (time.time() - t0), flush=True)
os.environ["H2G_VERBOSE"] = "1"
t0 = time.time()
ch = h2g.factorize(A, c["eps"], schedule=sched)
print("factorize wall %.1f s" % (time.time() - t0), ch.timing(), flush=True)
print([(l["level"], l["rank_sum_after"], l["eliminated"]) for l in ch.levels()], "root", ch.root_size, flush=True)
b = h2g.random_rhs(A.n, 1234) if hasattr(h2g, "random_rhs") else None
x = ch.solve(b)
print("residual (H2 matvec) %.3e" % A.relative_residual(x, b), "solve ms", ch.timing()["solve_ms"], flush=True)
