#!/bin/bash
# Round-2 GPU session O: Schur tile skipping 8x8 blocks outside the target, split solve records (row slabs): parity tests, solve timing per split threshold, per-level times, bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_gpu_hooks.py tests/test_gpu_cfg4a_parity.py tests/test_serialize.py -m gpu -q -x > gpurun_out/r02o_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02o_pytest.log
for sp in 0 256 128 96 64; do
  echo "H2G_SOLVE_SPLIT=$sp" >> gpurun_out/r02o_solve.log
  H2G_SOLVE_SPLIT=$sp timeout 600 python scripts/solve_only.py 2 >> gpurun_out/r02o_solve.log 2>&1
done
H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 > gpurun_out/r02o_prof_levels.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err; echo "bench rc $?" >> gpurun_out/r02o_bench.err
