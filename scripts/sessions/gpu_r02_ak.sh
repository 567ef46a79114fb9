#!/bin/bash
# Round-2 GPU session AK: Schur target / panel descriptors resolved once per batch (k_schur_resolve): tests, per-level Schur time with and without.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_gpu_dist.py tests/test_gpu_hooks.py -m gpu -q -x > gpurun_out/r02ak_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02ak_pytest.log
for r in 1 0 1 0; do
  echo "== H2G_SCHUR_RESOLVE=$r" >> gpurun_out/r02ak_prof.log
  H2G_SCHUR_RESOLVE=$r H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 2>&1 | grep -E " schur |factor_ms" >> gpurun_out/r02ak_prof.log
done
H2G_SCHUR_RESOLVE=1 timeout 300 python scripts/solve_only.py 2 > gpurun_out/r02ak_solve.log 2>&1
