#!/bin/bash
# Round-2 GPU session A: GPU tests, a short bench, and the config-2 golden
# oracle run on the GPU-built H² (oracle on the box's host cores).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
(nproc; lscpu | grep -E "Model name|Socket|Core|Thread"; free -g; nvidia-smi -L) > gpurun_out/r02a_host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02a_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02a_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc $?" >> gpurun_out/r02a_bench.err
timeout 3000 python scripts/oracle_golden.py 2 gpurun_out/golden/cfg2_oracle --h2 gpu > gpurun_out/golden/log.txt 2>&1; echo "golden rc $?" >> gpurun_out/golden/log.txt
