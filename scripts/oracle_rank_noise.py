"""Oracle self-noise at one BASELINE config (test infrastructure): the same
H² input factorized twice by the oracle, once with forward and once with
reversed GEMM inner-product order (two valid BLAS summation orders of the
same reference algorithm, proj/include/h2lu/factorization.hpp), comparing the
per-(level, cluster) rank_after. The result bounds how closely ANY
implementation can match the reference's ranks at this configuration.

usage: python scripts/oracle_rank_noise.py CONFIG OUT_JSON [H2_FILE [EPS]]
(H2_FILE: an H2LU matrix to factorize, e.g. the GPU-built input; default:
built by the oracle)"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import pyoracle as O  # noqa: E402
from helpers import vie_problem  # noqa: E402
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS  # noqa: E402

cfg, out = int(sys.argv[1]), sys.argv[2]
c = dict(BASELINE_CONFIGS[cfg])
if len(sys.argv) > 4:
    c["eps"] = float(sys.argv[4])
if len(sys.argv) > 3:
    A = O.load_h2(sys.argv[3])
else:
    A, K = vie_problem(c["cells"], c["side"], c["leaf"], c["eps"])
runs = {}
variants = [("forward", False, 0), ("reverse", True, 0)]
if os.environ.get("NOISE_GRAM"):
    variants.append(("gram", False, 1))  # the step-0 truncation through the Gram (paper Eq. 16-18)
for name, rev, mode in variants:
    O.set_gemm_order(rev)
    O.set_truncation(mode)
    t0 = time.time()
    ch = A.factorize(c["eps"])
    runs[name] = ({(r["level"], r["cluster"]): r["rank_after"] for r in ch.all_records()}, [l["rank_sum_after"] for l in ch.levels()],
                  ch.root_size, time.time() - t0)
    print(name, runs[name][1], runs[name][2], "%.0f s" % runs[name][3], flush=True)
O.set_gemm_order(False)
O.set_truncation(0)
rf, rr = runs["forward"][0], runs["reverse"][0]
d = {k: rr[k] - rf[k] for k in rf}
per_level = {}
for lv in sorted({k[0] for k in rf}, reverse=True):
    dl = np.array([v for k, v in d.items() if k[0] == lv])
    per_level[str(lv)] = dict(max_abs=int(np.abs(dl).max()), nonzero=int(np.count_nonzero(dl)), clusters=int(dl.size))
mean_abs = {}
for lv in sorted({k[0] for k in rf}, reverse=True):
    mean_abs[str(lv)] = float(np.mean([abs(v) for k, v in d.items() if k[0] == lv]))
res = dict(config=cfg, eps=c["eps"], mean_abs_per_level=mean_abs, perturbation="GEMM inner-product order reversed (oracle/dense.hpp gemm_acc); same H2 input",
           max_abs_rank_diff=int(max(abs(v) for v in d.values())), nonzero=int(sum(1 for v in d.values() if v)), clusters=len(d),
           per_level=per_level, rank_sum_after_forward=runs["forward"][1], rank_sum_after_reverse=runs["reverse"][1],
           root_forward=runs["forward"][2], root_reverse=runs["reverse"][2])
if "gram" in runs:
    rgm = runs["gram"][0]
    dg = {k: rgm[k] - rf[k] for k in rf}
    res["gram_variant"] = dict(perturbation="step-0 truncation through the Gram of the projected fill (paper Eq. 16-18) instead of QR + SVD",
                               max_abs_rank_diff=int(max(abs(v) for v in dg.values())),
                               per_level={str(lv): dict(max_abs=int(max(abs(v) for k, v in dg.items() if k[0] == lv)),
                                                       mean_abs=float(np.mean([abs(v) for k, v in dg.items() if k[0] == lv])))
                                          for lv in sorted({k[0] for k in rf}, reverse=True)},
                               rank_sum_after=runs["gram"][1], root=runs["gram"][2])
json.dump(res, open(out, "w"), indent=1)
keys = sorted(rf)
np.savez_compressed(os.path.splitext(out)[0] + ".npz", level_cluster=np.array(keys, np.int64), forward=np.array([rf[k] for k in keys], np.int64),
                    reverse=np.array([rr[k] for k in keys], np.int64))
print(json.dumps(res))
