#!/bin/bash
# Round-2 GPU session AJ: pinned staging buffers cached and reused: storage equality test, config 3 at eps 1e-4 again.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r02aj_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02aj_pytest.log
timeout 3000 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02aj_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02aj_cfg3_1e-4.log
