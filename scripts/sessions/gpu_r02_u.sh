#!/bin/bash
# Round-2 GPU session U: global-memory Gram fallback of the step-0 tridiagonalization, k-parallel many-RHS substitution GEMVs: tests, solve timing, config 3 at eps 1e-3.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_gpu_cfg4a_parity.py -m gpu -q -x > gpurun_out/r02u_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02u_pytest.log
timeout 600 python scripts/solve_only.py 2 > gpurun_out/r02u_solve.log 2>&1
timeout 2400 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02u_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02u_cfg3_1e-3.log
