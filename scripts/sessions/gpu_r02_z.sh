#!/bin/bash
# Round-2 GPU session Z: compute-sanitizer (memcheck, racecheck, synccheck) on the small case covering the cluster kernels, the dataflow solve with split records, the streamed chain and the SUBTREE order.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 600 python scripts/sanitize_case.py > gpurun_out/r02z_plain.log 2>&1 || { echo "plain run failed" >> gpurun_out/r02z_plain.log; exit 1; }
timeout 1800 $CS --tool memcheck --print-limit 30 python scripts/sanitize_case.py > gpurun_out/r02z_memcheck.log 2>&1; echo "memcheck rc $?" >> gpurun_out/r02z_memcheck.log
timeout 2400 $CS --tool racecheck --racecheck-report all --print-limit 30 python scripts/sanitize_case.py > gpurun_out/r02z_racecheck.log 2>&1; echo "racecheck rc $?" >> gpurun_out/r02z_racecheck.log
timeout 1800 $CS --tool synccheck --print-limit 30 python scripts/sanitize_case.py > gpurun_out/r02z_synccheck.log 2>&1; echo "synccheck rc $?" >> gpurun_out/r02z_synccheck.log
