#!/bin/bash
# Round-2 GPU session V: config 3 at its nominal eps 1e-4; config 4 (explicit inverse, 64 RHS) at eps 1e-3.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 3000 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02v_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02v_cfg3_1e-4.log
timeout 2400 python scripts/try_config.py 4 reference 1e-3 64 > gpurun_out/r02v_cfg4_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02v_cfg4_1e-3.log
