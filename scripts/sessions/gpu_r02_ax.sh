#!/bin/bash
# Round-2 GPU session AX: right-hand-side groups in waves (at most 16 groups, gathered-partials budget): parity tests, config-2 64-RHS and 256-RHS timing.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r02ax_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02ax_pytest.log
timeout 600 python scripts/solve_threads.py 2 150 > gpurun_out/r02ax_cfg2.log 2>&1
timeout 600 python scripts/many_rhs.py 2 256 >> gpurun_out/r02ax_cfg2.log 2>&1
