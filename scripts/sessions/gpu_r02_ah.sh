#!/bin/bash
# Round-2 GPU session AH: K-split width of the step-0 Gram partials (CTA count of the Gram GEMMs on small batches).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for w in 0 128 256 1024; do
  echo "== H2G_GRAM_PARTW=$w" >> gpurun_out/r02ah_prof.log
  H2G_GRAM_PARTW=$w H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 2>&1 | grep -E " gram | eig1 |factor_ms" >> gpurun_out/r02ah_prof.log
done
