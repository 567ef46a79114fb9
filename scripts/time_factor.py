"""Times one factorization of a BASELINE config with per-level host/device logs."""
import os
import sys
import time

sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g  # noqa: E402
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
c = BASELINE_CONFIGS[cfg]
k0, scale, diag = vie_constants(c["cells"], c["side"])
t0 = time.time()
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.helmholtz_kernel(k0, diag, scale), c["eps"])
print("build", time.time() - t0, flush=True)
for i in range(2):
    t0 = time.time()
    ch = h2g.factorize(A, c["eps"], schedule=sched)
    print("factorize wall", time.time() - t0, ch.timing(), flush=True)
print([(l["level"], l["rank_sum_after"], l["eliminated"]) for l in ch.levels()], ch.root_size)
A.ctx.set_profiling(True)
ch = h2g.factorize(A, c["eps"], schedule=sched)
print({k: (round(v["ms"], 1), v["launches"]) for k, v in ch.kernel_stats().items()})
print("work", ch.work())
