#!/bin/bash
# Round-2 GPU session AP: config 4 (262144 unknowns, 64 RHS, explicit inverse) with the right-hand-side groups side by side: eps 1e-2 and 1e-4.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02ap_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02ap_cfg4_1e-2.log
timeout 1500 python scripts/try_config.py 4 reference 1e-4 64 > gpurun_out/r02ap_cfg4_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02ap_cfg4_1e-4.log
