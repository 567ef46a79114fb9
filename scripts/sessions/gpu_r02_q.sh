#!/bin/bash
# Round-2 GPU session Q: lifted panels double-buffered per batch (memory), config 3 at eps 1e-3 again, bench under torchrun with 2 ranks on the one GPU (gloo exchange).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/r02q_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02q_pytest.log
timeout 1500 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02q_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02q_cfg3_1e-3.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29671 bench.py --gpus 2 --steps 2 --warmup 1 --no-e2e > gpurun_out/r02q_bench_2ranks.json 2> gpurun_out/r02q_bench_2ranks.err; echo "rc $?" >> gpurun_out/r02q_bench_2ranks.err
