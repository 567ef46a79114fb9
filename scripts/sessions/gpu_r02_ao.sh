#!/bin/bash
# Round-2 GPU session AO: step-0 refinement switch at eps = 1e-6 (Gram-only against refined against the oracle).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python scripts/refine_switch.py 1e-6 > gpurun_out/r02ao_refine_1e-6.log 2>&1; echo "exit $?" >> gpurun_out/r02ao_refine_1e-6.log
timeout 900 python scripts/refine_switch.py 1e-5 > gpurun_out/r02ao_refine_1e-5.log 2>&1; echo "exit $?" >> gpurun_out/r02ao_refine_1e-5.log
