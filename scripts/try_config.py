"""Build and factorize one BASELINE config with level logging; report ranks,
times and residuals (one JSON summary line at the end).

usage: python scripts/try_config.py CONFIG [SCHEDULE] [EPS] [NRHS] [explicit]
EPS overrides both eps_h2 and eps_fill (config 4's sweep); NRHS > 1 applies the
factorization to that many seeded RHS at once (seeds 1234 + c). Config 4 uses
the explicit-inverse application (h2g_solve mode APPLY_INVERSE_EXPLICIT)."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sched = sys.argv[2] if len(sys.argv) > 2 else "reference"
c = dict(BASELINE_CONFIGS[cfg])
if len(sys.argv) > 3:
    c["eps"] = float(sys.argv[3])
nrhs = int(sys.argv[4]) if len(sys.argv) > 4 else 1
k0, scale, diag = vie_constants(c["cells"], c["side"])
K = h2g.helmholtz_kernel(k0, diag, scale)
pts = vie_grid_points(c["cells"], c["side"])
t0 = time.time()
A = h2g.H2Matrix.build(pts, c["leaf"], 1.0, K, c["eps"])
build_s = time.time() - t0
print("config %d eps %.0e: N %d, build %.1f s" % (cfg, c["eps"], A.n, build_s), flush=True)
perm = A.perm()
os.environ.setdefault("H2G_VERBOSE", "1")
t0 = time.time()
ch = h2g.factorize(A, c["eps"], schedule=sched)
wall = time.time() - t0
tm = ch.timing()
print("factorize wall %.1f s" % wall, tm, flush=True)
levels = [(l["level"], l["rank_sum_before"], l["rank_sum_after"], l["eliminated"]) for l in ch.levels()]
recs = ch.all_records()
rmax = {}
for r in recs:
    rmax[r["level"]] = max(rmax.get(r["level"], 0), r["rank_after"])
print("levels (level, rank_sum_before, rank_sum_after, eliminated):", levels, "root", ch.root_size, flush=True)
if nrhs == 1:
    b = h2g.random_rhs(A.n, 1234)
else:
    b = np.stack([h2g.random_rhs(A.n, 1234 + j) for j in range(nrhs)], axis=1)
if perm is not None:
    b = b[perm]  # original order -> tree order
explicit = cfg == 4 or (len(sys.argv) > 5 and sys.argv[5] == "explicit")
mode = "apply_inverse_explicit" if explicit else "solve"
t0 = time.time()
x = ch.apply_inverse_explicit(b) if explicit else ch.solve(b)
solve_wall = time.time() - t0
solve_ms = ch.timing()["solve_ms"]
print("%s wall %.3f s, device ms %.2f" % (mode, solve_wall, solve_ms), flush=True)
cols = [0] if nrhs == 1 else list(range(0, nrhs, max(1, nrhs // 4)))
res_h2, res_d = [], []
pts_tree = pts[perm] if perm is not None else None
rng = np.random.default_rng(1234)
rows = np.sort(rng.choice(A.n, size=min(4096, A.n), replace=False)).astype(np.int64)
for j in cols:
    xj = x if nrhs == 1 else x[:, j]
    bj = b if nrhs == 1 else b[:, j]
    res_h2.append(A.relative_residual(xj, bj))
    if pts_tree is not None:
        res_d.append(h2g.sampled_dense_residual(pts_tree, K, xj, bj, rows))
print("relative residual (H2 matvec):", ["%.3e" % v for v in res_h2], "sampled dense rows:", ["%.3e" % v for v in res_d], flush=True)
print("SUMMARY " + json.dumps(dict(config=cfg, eps=c["eps"], n=A.n, schedule=sched, nrhs=nrhs, build_s=build_s, factor_ms=tm["factor_ms"],
                                   factor_wall_s=wall, plan_ms=tm["plan_ms"], solve_mode=mode, solve_ms=solve_ms, solve_wall_s=solve_wall,
                                   levels=levels, rank_max_per_level=rmax, root=ch.root_size, residual_h2=res_h2, residual_sampled_dense=res_d,
                                   residual_columns=cols)), flush=True)
