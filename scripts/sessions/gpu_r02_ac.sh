#!/bin/bash
# Round-2 GPU session AC: L2 prefetch of an item's chain data before its dependency wait (dataflow solve): tests and timing.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_serialize.py -m gpu -q -x > gpurun_out/r02ac_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02ac_pytest.log
timeout 600 python scripts/solve_only.py 2 > gpurun_out/r02ac_solve.log 2>&1
timeout 600 python scripts/solve_only.py 2 colored >> gpurun_out/r02ac_solve.log 2>&1
