#!/bin/bash
# Round-2 GPU session AV: one-thread-per-entry many-RHS paths at every size, 4 columns per thread: parity tests, config-2 timing, config 4 at eps 1e-2 with 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py -m gpu -q -x > gpurun_out/r02av_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02av_pytest.log
timeout 600 python scripts/solve_threads.py 2 150 100 > gpurun_out/r02av_cfg2.log 2>&1
H2G_SOLVE_SMALLK=0 timeout 600 python scripts/solve_threads.py 2 150 >> gpurun_out/r02av_cfg2.log 2>&1
timeout 900 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02av_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02av_cfg4_1e-2.log
