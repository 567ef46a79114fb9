#!/bin/bash
# Round-2 GPU session AA: Schur tile experiments on config 2 (per-level event times): 4 pipeline stages, 32x32 DFMA tiles on the fine levels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
run() {
  echo "== $*" >> gpurun_out/r02aa_prof.log
  env "$@" H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 2>&1 | grep -E "schur|factor_ms" >> gpurun_out/r02aa_prof.log
}
run H2G_SCHUR_STAGES=3
run H2G_SCHUR_STAGES=4
run H2G_SCHUR_T32_BMAX=64
run H2G_SCHUR_T32_BMAX=128
run H2G_SCHUR_T32_BMAX=64 H2G_SCHUR_STAGES=4
