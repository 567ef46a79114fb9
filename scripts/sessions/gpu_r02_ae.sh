#!/bin/bash
# Round-2 GPU session AE: config 4 (explicit inverse, 64 RHS) at eps 1e-4 and 1e-2 with the automatic settings (64 segments, default host staging cap).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 3000 python scripts/try_config.py 4 reference 1e-4 64 > gpurun_out/r02ae_cfg4_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02ae_cfg4_1e-4.log
timeout 1500 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02ae_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02ae_cfg4_1e-2.log
