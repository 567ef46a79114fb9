"""Factorize the same matrix several times; report chain hash and per-level rank sums."""
import sys
sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
for r in range(reps):
    ch = h2g.factorize(A, c["eps"], schedule=sched)
    print(r, hex(ch.hash()), [l["rank_sum_after"] for l in ch.levels()], ch.timing()["factor_ms"], flush=True)
    del ch
