#!/bin/bash
# Round-2 GPU session AZ: k-slices capped at k in the few-RHS substitution GEMVs: parity tests, solve timing on config 2.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_gpu_hooks.py -m gpu -q -x > gpurun_out/r02az_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02az_pytest.log
timeout 600 python scripts/solve_only.py 2 > gpurun_out/r02az_solve.log 2>&1
