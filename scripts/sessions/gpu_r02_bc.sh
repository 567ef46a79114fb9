#!/bin/bash
# Round-2 GPU session BC: config 4's eps sweep {1e-2, 1e-4, 1e-6} with 64 RHS through the explicit inverse on the 32^3 cube (the size at which every eps fits one B200).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02bc_sweep.log
for e in 1e-2 1e-4 1e-6; do
  H2G_VERBOSE=0 timeout 600 python scripts/try_config.py 2 reference $e 64 explicit 2>/dev/null | grep -E "^config|^factorize|^levels|^apply|^relative|^SUMMARY" >> gpurun_out/r02bc_sweep.log
done
