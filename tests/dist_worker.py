"""One rank of the multi-GPU subtree-partitioned factorization (launched by
torch.distributed.run from tests/test_gpu_dist.py and scripts): every rank
builds the same seeded H2 input with the oracle, uploads it to its GPU
(LOCAL_RANK modulo the visible device count, so world_size 2 also runs on one
GPU), runs h2g.factorize_dist and solves; rank 0 compares with the
single-process SUBTREE factorization and prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch
import torch.distributed as dist

import paper_1703_06155_b200 as h2g
from helpers import vie_problem


def main():
    cells, side, leaf, eps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
    ndev = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = local % ndev
    torch.cuda.set_device(dev)
    # NCCL needs one GPU per rank; ranks sharing a GPU (tests) exchange through gloo
    backend = "nccl" if ndev >= int(os.environ["WORLD_SIZE"]) else "gloo"
    dist.init_process_group(backend)
    me, n = dist.get_rank(), dist.get_world_size()
    ctx = h2g.Context(dev)
    if len(sys.argv) > 5 and sys.argv[5] == "gpu-build":
        # large cases: the H2 is built on every rank's device (same seeded input, same result)
        from paper_1703_06155_b200.geometry import vie_grid_points

        G = h2g.H2Matrix.build(vie_grid_points(cells, side), leaf, 1.0, h2g.vie_kernel(cells, side), eps, ctx)
    else:
        A, _ = vie_problem(cells, side, leaf, eps)
        G = h2g.H2Matrix.upload(A.arrays(), ctx)
    ch = h2g.factorize_dist(G, eps)
    b = h2g.random_rhs(G.n, 1234)
    x = ch.solve(b)
    st = ch.dist_stats()
    hashes = [None] * n
    dist.all_gather_object(hashes, ch.hash())
    if me == 0:
        ref = h2g.factorize(G, eps, schedule="subtree")
        xr = ref.solve(b)
        print("DIST " + json.dumps(dict(backend=backend, nranks=n, hashes=[str(h) for h in hashes], single_hash=str(ref.hash()),
                                        x_equal=bool(np.array_equal(x, xr)), residual=G.relative_residual(x, b),
                                        sent_bytes=st["sent_bytes"], total_bytes=st["total_bytes"], exchange_s=st["exchange_s"],
                                        factor_ms=ch.timing()["factor_ms"], single_factor_ms=ref.timing()["factor_ms"])), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
