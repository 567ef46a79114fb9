"""Steady-state host/device phase timing of one factorize (H2G_VERBOSE=2 on the 2nd call)."""
import os, sys
sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"], schedule=sched)
print("cold", ch.timing(), flush=True)
del ch
ch = h2g.factorize(A, c["eps"], schedule=sched)
print("warm", ch.timing(), flush=True)
del ch
os.environ["H2G_VERBOSE"] = sys.argv[3] if len(sys.argv) > 3 else "2"
ch = h2g.factorize(A, c["eps"], schedule=sched)
print("warm verbose", ch.timing(), flush=True)
