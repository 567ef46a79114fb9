#!/bin/bash
# Round-2 GPU session P: multi-GPU subtree partition (2 and 4 ranks sharing the box's GPU, gloo exchange) against the single-process SUBTREE run; config-2 partitioned run.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x > gpurun_out/r02p_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02p_pytest.log
H2G_VERBOSE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29655 tests/dist_worker.py 32 1.0 32 1e-4 gpu-build > gpurun_out/r02p_dist_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/r02p_dist_cfg2.log
