#!/bin/bash
# Round-2 GPU session BD: the eps = 1e-6 cube test.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cfg2_parity.py -m gpu -q -x --durations=5 > gpurun_out/r02bd_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02bd_pytest.log
