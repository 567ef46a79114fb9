#!/bin/bash
# Round-2 GPU session AT: one thread per result entry for short inner dimensions in the many-RHS paths (fine levels): parity tests, 64-RHS timing.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py -m gpu -q -x > gpurun_out/r02at_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02at_pytest.log
timeout 600 python scripts/solve_groups.py 2 > gpurun_out/r02at_groups_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/r02at_groups_cfg2.log
