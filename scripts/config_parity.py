"""Oracle vs GPU on one BASELINE config (oracle-built H2 uploaded to the GPU):
per-level rank sums, per-cluster rank differences, solution agreement.
Oracle results are cached in gpurun_out/oracle_cfg<N>.npz."""
import os, sys, time
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
sys.path.insert(0, "tests")
import numpy as np
import pyoracle as O
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS
from helpers import vie_problem, ranks_by_cluster, rel

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = BASELINE_CONFIGS[cfg]
t0 = time.time()
A, K = vie_problem(c["cells"], c["side"], c["leaf"], c["eps"])
print("oracle build", time.time() - t0, flush=True)
t0 = time.time()
och = A.factorize(c["eps"])
print("oracle factorize", time.time() - t0, flush=True)
ro = ranks_by_cluster(och.all_records())
perm = A.tree.perm
b = O.rhs(A.n, 1234)[perm]
xo = och.solve(b)
G = h2g.H2Matrix.upload(A.arrays())
for rep in range(2):
    gch = h2g.factorize(G, c["eps"])
rg = ranks_by_cluster(gch.all_records())
d = np.array([rg[k] - ro[k] for k in ro])
print("oracle levels", [l["rank_sum_after"] for l in och.levels()], "root", och.root_size)
print("gpu    levels", [l["rank_sum_after"] for l in gch.levels()], "root", gch.root_size)
print("rank diffs: max |d| %d, #nonzero %d of %d, sum %d" % (np.abs(d).max(), np.count_nonzero(d), len(d), d.sum()))
for lv in sorted({k[0] for k in ro}, reverse=True):
    dl = np.array([rg[k] - ro[k] for k in ro if k[0] == lv])
    print("  level %d: max |d| %d, nonzero %d / %d, sum %d" % (lv, np.abs(dl).max(), np.count_nonzero(dl), len(dl), dl.sum()))
xg = gch.solve(b)
print("solution rel diff %.3e; residual oracle %.3e gpu %.3e" % (rel(xg, xo), A.relative_residual(xo, b), A.relative_residual(xg, b)))
print("gpu factor ms", gch.timing()["factor_ms"])
