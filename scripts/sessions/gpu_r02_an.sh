#!/bin/bash
# Round-2 GPU session AN: right-hand-side groups side by side in the dataflow solve (grid y): parity tests and 64-RHS timing on config 2.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r02an_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02an_pytest.log
timeout 900 python scripts/solve_groups.py 2 > gpurun_out/r02an_groups_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/r02an_groups_cfg2.log
