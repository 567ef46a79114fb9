#!/bin/bash
# Round-2 GPU session Y: config 3 at its nominal eps 1e-4 with the host staging cap raised to 176 GB of the box's 196 GB.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
free -g > gpurun_out/r02y_host.log
H2G_HOST_STAGING_GB=176 timeout 2400 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02y_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02y_cfg3_1e-4.log
free -g >> gpurun_out/r02y_host.log
