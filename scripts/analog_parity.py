"""GPU vs the committed oracle run on a scaled analog of a large config
(same spacing h, leaf and eps, fewer cells): ranks per level, solution and
residuals (used for the config-4 geometry at eps 1e-2, where the full
262144-unknown problem has no CPU oracle run).

usage: python scripts/analog_parity.py GOLDEN_PREFIX"""
import json
import sys

sys.path[:0] = [".", "tests", "oracle"]
import numpy as np

import paper_1703_06155_b200 as h2g
from helpers import h2_input_hash, rel, sampled_rows
from paper_1703_06155_b200.geometry import vie_constants, vie_grid_points

pre = sys.argv[1]
meta = json.load(open(pre + ".json"))
gold = np.load(pre + ".npz")
k0, scale, diag = vie_constants(meta["cells"], meta["side"])
pts = vie_grid_points(meta["cells"], meta["side"])
K = h2g.helmholtz_kernel(k0, diag, scale)
A = h2g.H2Matrix.build(pts, meta["leaf"], 1.0, K, meta["eps"])
host = A.download()
same = h2_input_hash(host) == meta["input_sha256"]
ch = h2g.factorize(A, meta["eps"])
perm = host["perm"]
b = h2g.random_rhs(A.n, 1234)[perm]
x = ch.solve(b)
rows = sampled_rows(A.n)
r_h2 = A.relative_residual(x, b)
r_d = h2g.sampled_dense_residual(pts[perm], K, x, b, rows)
ro = {(int(r[0]), int(r[1])): int(r[4]) for r in gold["rec"]}
rg = {(r["level"], r["cluster"]): r["rank_after"] for r in ch.all_records()}
out = dict(identical_input=same, n=A.n, eps=meta["eps"], x_rel_diff=rel(x, gold["x"]), residual_h2=[r_h2, meta["residual_h2"]],
           residual_sampled_dense=[r_d, meta["residual_sampled_dense"]], levels={})
for lv in sorted({k[0] for k in ro}, reverse=True):
    d = np.array([rg[k] - ro[k] for k in ro if k[0] == lv])
    out["levels"][lv] = dict(max_abs=int(np.abs(d).max()), mean_abs=float(np.abs(d).mean()), sum_gpu=int(sum(v for k, v in rg.items() if k[0] == lv)),
                             sum_oracle=int(sum(v for k, v in ro.items() if k[0] == lv)))
print(json.dumps(out))
