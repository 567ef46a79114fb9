#!/bin/bash
# Round-2 GPU session AR: CTA width x shared-memory budget of the grouped 64-RHS dataflow solve (config 2).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02ar_threads.log
for t in 256 512 1024; do
  H2G_SOLVE_THREADS=$t timeout 600 python scripts/solve_threads.py 2 200 150 100 64 48 >> gpurun_out/r02ar_threads.log 2>&1
done
