#!/bin/bash
# Round-2 GPU session AM: eps = 1e-6 — the config-2 geometry with 64 RHS (explicit inverse), then the config-4 attempt (memory record).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python scripts/try_config.py 2 reference 1e-6 64 explicit > gpurun_out/r02am_cfg2geom_1e-6.log 2>&1; echo "exit $?" >> gpurun_out/r02am_cfg2geom_1e-6.log
timeout 1800 python scripts/try_config.py 4 reference 1e-6 64 > gpurun_out/r02am_cfg4_1e-6.log 2>&1; echo "exit $?" >> gpurun_out/r02am_cfg4_1e-6.log
nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/r02am_cfg4_1e-6.log 2>&1
