"""Host-side logic of the multi-GPU subtree partition (h2g_factorize_dist,
north_star / SURVEY §8e option 2), checked without a GPU: the SUBTREE schedule
and the per-subtree exchange lists (h2g_partition_plan), and the exchange
callback over torch.distributed with world_size 2 (gloo)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1703_06155_b200 as h2g
from helpers import vie_problem

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cube_arrays():
    # 16^3 grid, leaf 8: 512 leaf clusters, 64 per level-3 subtree; a loose H2
    # tolerance keeps the build short (only the structure matters here)
    A, _ = vie_problem(16, 0.5, 8, 1e-1)
    return A.arrays()


def test_subtree_schedule_and_exchange_lists(cube_arrays):
    depth = int(np.asarray(cube_arrays["depth"]).reshape(-1)[0])
    seen_interior = 0
    for level in range(depth, 4, -1):
        pp = h2g.partition_plan(cube_arrays, level)
        nl, pb = pp["nl"], pp["part_batch"]
        shift = level - 3
        sub = np.arange(nl) >> shift
        # neighbours from the dense blocks
        r, c = pp["dense_rc"][:, 0], pp["dense_rc"][:, 1]
        off = r != c
        crosses = np.zeros(nl, bool)
        np.logical_or.at(crosses, r[off], sub[r[off]] != sub[c[off]])
        interior = ~crosses
        bo = pp["batch_of"]
        # every cluster has a batch; interior clusters sit in their own subtree's batch range, boundary clusters after all of them
        assert bo.min() >= 0 and bo.max() == pp["batches"] - 1
        assert np.all(np.diff(pb) >= 0)
        for t in range(nl):
            if interior[t]:
                assert pb[sub[t]] <= bo[t] < pb[sub[t] + 1], (level, t)
            else:
                assert bo[t] >= pb[8], (level, t)
        # dense neighbours never share a batch, and a lower-id neighbour of the same group comes first
        assert np.all(bo[r[off]] != bo[c[off]])
        same_group = interior[r] == interior[c]
        lower = off & same_group & (c < r)
        assert np.all(bo[c[lower]] < bo[r[lower]])
        # exchange lists: no block is written by two subtrees, and what a subtree's interior phase writes lies inside the subtree
        for part, rc in ((pp["dense_part"], pp["dense_rc"]), (pp["fill_part"], pp["fill_rc"])):
            assert not np.any(part == -2)
            w = part >= 0
            assert np.all(sub[rc[w, 0]] == part[w]) and np.all(sub[rc[w, 1]] == part[w])
        # every block an interior cluster touches directly (its row and column) is on its subtree's list
        touched = interior[r] | interior[c]
        assert np.all(pp["dense_part"][touched] >= 0)
        seen_interior += int(interior.sum())
    assert seen_interior > 100  # the fixture has real interiors (216 of 512 leaves)


_WORKER = r'''
import sys
sys.path.insert(0, %(root)r)
import numpy as np, ctypes as C
import torch.distributed as dist
import paper_1703_06155_b200 as h2g
dist.init_process_group("gloo")
me, n = dist.get_rank(), dist.get_world_size()
# uneven parts, one of them empty on the second round
for sizes in ([1000, 24], [0, 4096], [64, 0]):
    offs = np.zeros(n + 1, np.int64)
    offs[1:] = np.cumsum(sizes)
    buf = np.full(int(offs[-1]), 255, np.uint8)
    buf[offs[me]:offs[me + 1]] = (np.arange(sizes[me]) * (me + 3) + me) %% 251
    errors = []
    ex = h2g.torch_exchange(None, device_buffers=False, errors=errors)
    rc = ex(buf.ctypes.data, offs.ctypes.data_as(C.POINTER(C.c_int64)), n)
    assert rc == 0 and not errors, errors
    for r in range(n):
        want = (np.arange(sizes[r]) * (r + 3) + r) %% 251
        assert np.array_equal(buf[offs[r]:offs[r + 1]], want.astype(np.uint8)), (me, r)
# a wrong rank count is reported, not swallowed
errors = []
ex = h2g.torch_exchange(None, device_buffers=False, errors=errors)
offs = np.zeros(4, np.int64)
assert ex(0, offs.ctypes.data_as(C.POINTER(C.c_int64)), 3) == 1 and errors
dist.barrier()
if me == 0:
    print("EXCHANGE OK")
dist.destroy_process_group()
'''


def test_exchange_callback_world2_gloo(tmp_path):
    path = str(tmp_path / "xchg_worker.py")
    open(path, "w").write(_WORKER % dict(root=ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29631", path]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert out.returncode == 0, out.stderr[-3000:]
    assert "EXCHANGE OK" in out.stdout
