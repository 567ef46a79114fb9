#!/bin/bash
# Round-2 GPU session W: chain levels return to HBM after the factorization: tests, config 4 at eps 1e-2 with 64 RHS, config 3 at eps 1e-3.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_serialize.py -m gpu -q -x > gpurun_out/r02w_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02w_pytest.log
timeout 1500 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02w_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02w_cfg4_1e-2.log
timeout 2400 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02w_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02w_cfg3_1e-3.log
