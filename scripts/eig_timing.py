"""One warm factorize with H2G_DEBUG=8 (k_eig1c phase timers)."""
import os, sys
sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
c = BASELINE_CONFIGS[2]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
del ch
os.environ["H2G_DEBUG"] = "8"
ch = h2g.factorize(A, c["eps"])
