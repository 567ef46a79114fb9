#!/bin/bash
# Round-2 GPU session AF: right-hand sides per pass of the dataflow solve (shared-memory budget) at 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for kb in 96 150 200; do
  echo "H2G_SOLVE_SMEM_KB=$kb" >> gpurun_out/r02af_solve.log
  H2G_SOLVE_SMEM_KB=$kb timeout 600 python scripts/solve_only.py 2 >> gpurun_out/r02af_solve.log 2>&1
done
