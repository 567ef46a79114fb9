#!/bin/bash
# Round-2 GPU session AD: config 3 at its nominal eps 1e-4 with 64 fill / chain segments per level (smaller chain halves and front pool) and the host staging cap at 176 GB.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
H2G_FILL_SEGMENTS=64 H2G_HOST_STAGING_GB=176 timeout 3000 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02ad_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02ad_cfg3_1e-4.log
free -g > gpurun_out/r02ad_host.log
