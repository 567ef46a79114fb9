"""Multi-GPU subtree partition (h2g_factorize_dist, SURVEY §8e option 2) on the
device: the SUBTREE order against the oracle run in the same sequential order,
and a world_size-2 run (two ranks sharing the one GPU of the test box, exchange
staged through gloo) that must reproduce the single-process SUBTREE
factorization bit for bit."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
import pyoracle as O
from helpers import ranks_by_cluster, rel, vie_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

# 16^3 grid with leaf 8: 512 leaves, 216 of them interior to a level-3 subtree
CUBE = (16, 0.5, 8, 1e-3)


def test_subtree_order_matches_oracle_interior_first():
    A, _ = vie_problem(*CUBE)
    eps = CUBE[3]
    # the SUBTREE batches are the wavefronts of the oracle's interior-first sequence (interior clusters ascending = subtree by subtree)
    och = A.factorize(eps, schedule=O.SCHEDULE_INTERIOR_FIRST)
    G = h2g.H2Matrix.upload(A.arrays())
    gch = h2g.factorize(G, eps, schedule="subtree")
    b = O.rhs(G.n, 5)
    xo, xg = och.solve(b), gch.solve(b)
    assert rel(xg, xo) <= 10 * eps
    ro, rg = ranks_by_cluster(och.all_records()), ranks_by_cluster(gch.all_records())
    assert ro.keys() == rg.keys()
    leaf_level = max(k[0] for k in ro)
    assert max(abs(ro[k] - rg[k]) for k in ro if k[0] == leaf_level) <= 1
    assert G.relative_residual(xg, b) <= 2 * A.relative_residual(xo, b) + 1e-12


def test_single_rank_dist_equals_subtree_schedule():
    A, _ = vie_problem(*CUBE)
    G = h2g.H2Matrix.upload(A.arrays())
    a = h2g.factorize(G, CUBE[3], schedule="subtree")
    b = h2g.factorize_dist(G, CUBE[3], rank=0, nranks=1)
    assert a.hash() == b.hash()
    with pytest.raises(h2g.InvalidInputError):
        h2g.factorize_dist(G, CUBE[3], rank=0, nranks=3, exchange=lambda *a: 0)


@pytest.mark.parametrize("nranks", [2, 4])
def test_partitioned_factorization_world_n_bitwise(nranks):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}", "--master-addr=127.0.0.1",
           f"--master-port={29640 + nranks}", os.path.join(ROOT, "tests", "dist_worker.py")] + [str(v) for v in CUBE]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])
    line = [l for l in out.stdout.splitlines() if l.startswith("DIST ")]
    assert len(line) == 1, out.stdout
    rec = json.loads(line[0][5:])
    assert rec["nranks"] == nranks
    assert len(set(rec["hashes"])) == 1, rec  # every rank ends with the same chain
    assert rec["hashes"][0] == rec["single_hash"], rec  # ... which is the single-GPU SUBTREE chain, bit for bit
    assert rec["x_equal"] and rec["residual"] < 1e-2
    assert rec["total_bytes"] > 0 and 0 < rec["sent_bytes"] < rec["total_bytes"]
