#!/bin/bash
# Round-2 GPU session AU: threshold of the one-thread-per-entry many-RHS paths (H2G_SOLVE_SMALLK) on config 2.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02au_smallk.log
for k in 0 32 64 128 256 512; do
  echo "H2G_SOLVE_SMALLK=$k" >> gpurun_out/r02au_smallk.log
  H2G_SOLVE_SMALLK=$k timeout 600 python scripts/solve_threads.py 2 150 100 >> gpurun_out/r02au_smallk.log 2>&1
done
