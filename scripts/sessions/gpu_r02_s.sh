#!/bin/bash
# Round-2 GPU session S: streamed chain arena (segments to pinned host memory): equality test, config 3 at eps 1e-3 and 1e-4.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_serialize.py tests/test_gpu_dist.py -m gpu -q -x > gpurun_out/r02s_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02s_pytest.log
free -g > gpurun_out/r02s_host.log; nproc >> gpurun_out/r02s_host.log
timeout 1800 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02s_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02s_cfg3_1e-3.log
timeout 2400 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02s_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02s_cfg3_1e-4.log
