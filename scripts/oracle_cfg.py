"""Run the CPU oracle on one BASELINE config (oracle build + factorize + solve)
and save per-cluster ranks, level stats and the solution for seed 1234 to an
npz, so GPU runs can be compared without re-running the (serial) oracle."""
import sys, time
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
sys.path.insert(0, "tests")
import numpy as np
import pyoracle as O
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS
from helpers import vie_problem

cfg, out = int(sys.argv[1]), sys.argv[2]
c = BASELINE_CONFIGS[cfg]
t0 = time.time()
A, K = vie_problem(c["cells"], c["side"], c["leaf"], c["eps"])
tb = time.time() - t0
t0 = time.time()
och = A.factorize(c["eps"])
tf = time.time() - t0
recs = och.all_records()
perm = A.tree.perm
b = O.rhs(A.n, 1234)[perm]
xo = och.solve(b)
res = A.relative_residual(xo, b)
np.savez(out, rec=np.array([[r["level"], r["cluster"], r["bsize"], r["rank_before"], r["rank_after"], r["eliminated"]] for r in recs]),
         levels=np.array([[l["level"], l["rank_sum_after"], l["eliminated"]] for l in och.levels()]), x=xo, residual=res,
         root=och.root_size, build_s=tb, factor_s=tf)
print("oracle cfg", cfg, "build %.1f s factorize %.1f s residual %.3e" % (tb, tf, res), [l["rank_sum_after"] for l in och.levels()])
