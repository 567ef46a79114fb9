"""Golden oracle run on one BASELINE config (test infrastructure).

Runs the CPU oracle (oracle/, the reference-order restatement of
proj/include/h2lu/factorization.hpp and solve.hpp) once and writes what the
GPU parity test compares against:

  * the SHA-256 of the H² input the oracle factorized (tree ranges, block
    lists, bases, couplings, dense blocks), so the GPU test can prove it
    factorizes the identical matrix;
  * per-(level, cluster) rank_after / eliminated, the level diagnostics and
    the root size;
  * x for the seeded RHS (mt19937_64(1234) + normal_distribution, original
    order, permuted to tree order) and both residuals: through the H²
    operator (verify.hpp:14-19) and on 4096 seeded sampled rows of the dense
    kernel;
  * the oracle's measured factorization time, thread count, nproc and CPU
    model.

  --h2 gpu     build the H² with the GPU builder (h2g_matrix_build, the
               benched input), download it and factorize that on the CPU
               (run on the GPU box; this is how tests/golden/ is produced)
  --h2 oracle  build the H² with the oracle's own CPU builder

Usage: python scripts/oracle_golden.py CONFIG OUT_PREFIX [--h2 gpu|oracle]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import pyoracle as O  # noqa: E402
from helpers import h2_input_hash, sampled_rows  # noqa: E402
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_constants, vie_grid_points  # noqa: E402


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("out")
    ap.add_argument("--h2", choices=["gpu", "oracle"], default="gpu")
    ap.add_argument("--eps", type=float, default=None)
    ap.add_argument("--cells", type=int, default=None, help="override: cells per side (a scaled analog of the config)")
    ap.add_argument("--side", type=float, default=None, help="override: cube side in wavelengths")
    args = ap.parse_args()
    c = dict(BASELINE_CONFIGS[args.config])
    if args.cells:
        c["cells"] = args.cells
    if args.side:
        c["side"] = args.side
    eps = args.eps or c["eps"]
    k0, scale, diag = vie_constants(c["cells"], c["side"])
    pts = vie_grid_points(c["cells"], c["side"])
    K = O.helmholtz(k0, diag, scale)
    tree = O.Tree(pts, c["leaf"])
    blocks = O.Blocks(tree, 1.0)
    t0 = time.time()
    if args.h2 == "gpu":
        import paper_1703_06155_b200 as h2g

        G = h2g.H2Matrix.build(pts, c["leaf"], 1.0, h2g.vie_kernel(c["cells"], c["side"]), eps)
        arr = G.download()
        ob, oe = tree.ranges()
        assert np.array_equal(arr["cluster_begin"], ob) and np.array_equal(arr["cluster_end"], oe), "GPU tree differs from the oracle tree"
        A = O.H2.from_arrays(blocks, eps, arr, K)
        del G
    else:
        A = O.H2(blocks, K, eps)
        arr = A.arrays()
    t_build = time.time() - t0
    digest = h2_input_hash(arr)
    print(f"[golden] cfg {args.config} H2 ({args.h2}) built in {t_build:.1f}s sha256 {digest[:16]}", flush=True)

    t0 = time.time()
    ch = A.factorize(eps)
    t_factor = time.time() - t0
    print(f"[golden] oracle factorize {t_factor:.1f}s", flush=True)
    recs = ch.all_records()
    n = A.n
    perm = tree.perm
    b = O.rhs(n, 1234)[perm]
    t0 = time.time()
    x = ch.solve(b)
    t_solve = time.time() - t0
    res_h2 = A.relative_residual(x, b)
    rows = sampled_rows(n)
    zx = tree.kernel_rows_matvec(K, rows, x)
    res_dense = float(np.linalg.norm(zx - b[rows]) / np.linalg.norm(b[rows]))
    np.savez_compressed(
        args.out + ".npz",
        rec=np.array([[r["level"], r["cluster"], r["bsize"], r["rank_before"], r["rank_after"], r["eliminated"]] for r in recs], np.int64),
        levels=np.array([[l["level"], l["rank_sum_before"], l["rank_sum_after"], l["eliminated"], l["ledger_blocks"]] for l in ch.levels()], np.int64),
        x=x,
    )
    meta = dict(
        config=args.config,
        cells=c["cells"],
        side=c["side"],
        n=n,
        leaf=c["leaf"],
        eps=eps,
        h2_source=args.h2,
        input_sha256=digest,
        schedule="reference (ascending heap id, factorization.hpp:618)",
        gemm_order=os.environ.get("H2O_GEMM_ORDER", "forward"),
        root_size=int(ch.root_size),
        rank_sum_after=[int(l["rank_sum_after"]) for l in ch.levels()],
        residual_h2=res_h2,
        residual_sampled_dense=res_dense,
        sampled_rows=int(rows.size),
        rhs="mt19937_64(1234) + normal_distribution, original order, permuted to tree order",
        oracle_factor_s=t_factor,
        oracle_solve_s=t_solve,
        h2_build_s=t_build,
        oracle_threads=int(os.environ.get("H2O_THREADS", "0")) or os.cpu_count(),
        nproc=os.cpu_count(),
        cpu_model=cpu_model(),
        host=platform.node(),
        when=time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    )
    json.dump(meta, open(args.out + ".json", "w"), indent=1)
    print("[golden]", json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
