"""Build and factorize one BASELINE config with level logging; report ranks, time, residual.

usage: python scripts/try_config.py CONFIG [SCHEDULE] [EPS] [NRHS]
EPS overrides both eps_h2 and eps_fill (config 4's sweep); NRHS > 1 applies the
factorization to that many seeded RHS at once (seeds 1234 + c)."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
c = dict(BASELINE_CONFIGS[cfg])
if len(sys.argv) > 3:
    c["eps"] = float(sys.argv[3])
nrhs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
k0, scale, diag = vie_constants(c["cells"], c["side"])
t0 = time.time()
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
print("config %d eps %.0e: N %d, build %.1f s" % (cfg, c["eps"], A.n, time.time() - t0), flush=True)
os.environ.setdefault("H2G_VERBOSE", "1")
t0 = time.time()
ch = h2g.factorize(A, c["eps"], schedule=sched)
print("factorize wall %.1f s" % (time.time() - t0), ch.timing(), flush=True)
print("levels (level, rank_sum_after, eliminated):", [(l["level"], l["rank_sum_after"], l["eliminated"]) for l in ch.levels()], "root", ch.root_size, flush=True)
if nrhs == 1:
    b = h2g.random_rhs(A.n, 1234)
else:
    b = np.stack([h2g.random_rhs(A.n, 1234 + j) for j in range(nrhs)], axis=1)
t0 = time.time()
x = ch.apply_inverse_explicit(b) if cfg == 4 else ch.solve(b)  # config 4: explicit-inverse application
print("solve wall %.3f s" % (time.time() - t0), "device solve ms", ch.timing()["solve_ms"], flush=True)
if nrhs == 1:
    print("relative residual (H2 matvec) %.3e" % A.relative_residual(x, b), flush=True)
else:
    r = [A.relative_residual(x[:, j], b[:, j]) for j in range(0, nrhs, max(1, nrhs // 4))]
    print("relative residual (H2 matvec), sampled columns:", ["%.3e" % v for v in r], flush=True)
