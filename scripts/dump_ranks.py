"""Per-cluster final ranks of one factorize (GPU-built config), saved to an npz."""
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points
cfg, out = int(sys.argv[1]), sys.argv[2]
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
ch = h2g.factorize(A, c["eps"])
recs = ch.all_records()
np.savez(out, rec=np.array([[r["level"], r["cluster"], r["bsize"], r["rank_before"], r["rank_after"], r["eliminated"]] for r in recs]))
print("saved", out, len(recs))
