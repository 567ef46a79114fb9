"""Per-level, per-kernel-class device time of one warm factorize (H2G_VERBOSE=1 for the table)."""
import os, sys
sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
verbose = os.environ.pop("H2G_VERBOSE", None)
ch = h2g.factorize(A, c["eps"], schedule=sched)  # warm-up (plan, pools)
del ch
if verbose:
    os.environ["H2G_VERBOSE"] = verbose
A.ctx.set_profiling(True)
ch = h2g.factorize(A, c["eps"], schedule=sched)
print(ch.timing())
