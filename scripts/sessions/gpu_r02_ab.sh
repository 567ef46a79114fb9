#!/bin/bash
# Round-2 GPU session AB: pull-mode forward updates on the fine levels: tests, solve timing per threshold; then the sanitizer runs of session Z.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_serialize.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/r02ab_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02ab_pytest.log
for pl in 0 32 64 128; do
  echo "H2G_SOLVE_PULL=$pl" >> gpurun_out/r02ab_solve.log
  H2G_SOLVE_PULL=$pl timeout 600 python scripts/solve_only.py 2 >> gpurun_out/r02ab_solve.log 2>&1
done
bash scripts/sessions/gpu_r02_z.sh
