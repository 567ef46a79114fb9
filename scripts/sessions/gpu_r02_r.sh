#!/bin/bash
# Round-2 GPU session R: level-entry memory breakdown of config 3 at eps 1e-3, bench with the per-level Schur roofline.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02r_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02r_cfg3_1e-3.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench rc $?" >> gpurun_out/r02r_bench.err
