"""The config-4 geometry (spacing h = 1/16, leaf 64) at eps = 1e-2 — the
accuracy at which the 262144-unknown cube runs on one B200 — on a 32^3 analog
(side 2 lambda, N = 32768) against a committed oracle run on the identical
GPU-built input (tests/golden/cfg4a_eps1e-2.*, scripts/oracle_golden.py
--cells 32 --side 2.0 --eps 1e-2): the CPU oracle cannot run the full cube
(SURVEY §8d), so this is the oracle counterpart of the config-4 residuals."""
import json
import os

import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
from helpers import h2_input_hash, rel, sampled_rows
from paper_1703_06155_b200.geometry import vie_constants, vie_grid_points

pytestmark = pytest.mark.gpu

PRE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg4a_eps1e-2")


def test_config4_geometry_eps1e2_against_oracle():
    meta = json.load(open(PRE + ".json"))
    gold = np.load(PRE + ".npz")
    eps = meta["eps"]
    k0, scale, diag = vie_constants(meta["cells"], meta["side"])
    pts = vie_grid_points(meta["cells"], meta["side"])
    K = h2g.helmholtz_kernel(k0, diag, scale)
    A = h2g.H2Matrix.build(pts, meta["leaf"], 1.0, K, eps)
    host = A.download()
    assert h2_input_hash(host) == meta["input_sha256"]
    ch = h2g.factorize(A, eps)
    perm = host["perm"]
    b = h2g.random_rhs(A.n, 1234)[perm]
    x = ch.solve(b)
    assert rel(x, gold["x"]) <= 10 * eps
    assert A.relative_residual(x, b) <= 2 * meta["residual_h2"]
    rows = sampled_rows(A.n)
    assert h2g.sampled_dense_residual(pts[perm], K, x, b, rows) <= 2 * meta["residual_sampled_dense"]
    # ranks: bounded by the oracle's own rank noise on this input
    # (tests/golden/cfg4a_rank_noise.json, GEMM order reversed): measured GPU
    # mean |d| 1.9 / 4.4 / 6.7 at levels 8 / 7 / 6 against the oracle's 2.1 /
    # 4.2 / 6.9 (max 26 / 20 / 21 against 20 / 14 / 16); the leaf level is
    # within the north_star's +-1 except where the oracle itself moves
    noise = json.load(open(os.path.join(os.path.dirname(PRE), "cfg4a_rank_noise.json")))
    ro = {(int(r[0]), int(r[1])): int(r[4]) for r in gold["rec"]}
    rg = {(r["level"], r["cluster"]): r["rank_after"] for r in ch.all_records()}
    assert ro.keys() == rg.keys()
    for lv in sorted({k[0] for k in ro}, reverse=True):
        d = np.array([rg[k] - ro[k] for k in ro if k[0] == lv])
        nz, nmean = noise["per_level"][str(lv)], noise["mean_abs_per_level"][str(lv)]
        assert np.abs(d).max() <= max(2, 2.5 * nz["max_abs"] + 1), (lv, np.abs(d).max(), nz)
        assert np.abs(d).mean() <= 5.0 * nmean + 1.0, (lv, np.abs(d).mean(), nmean)
        so = sum(v for k, v in ro.items() if k[0] == lv)
        sg = sum(v for k, v in rg.items() if k[0] == lv)
        assert abs(sg - so) <= 0.25 * so + 1, (lv, sg, so)
