"""Factorize config N once, then run the solve (for profiling the substitution kernels)."""
import sys
sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
b = h2g.random_rhs(A.n, 1234)
for _ in range(2):
    x = ch.solve(b)
print("solve ms", ch.timing()["solve_ms"])
