#!/bin/bash
# Round-2 GPU session N: concatenated Schur pipeline + wide solve CTAs: parity tests, solve timing per CTA width, per-level times, bench, config 3 at eps 1e-3.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_gpu_hooks.py tests/test_gpu_cfg4a_parity.py -q -x > gpurun_out/r02n_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02n_pytest.log
for nt in 256 512 1024 0; do
  echo "H2G_SOLVE_THREADS=$nt" >> gpurun_out/r02n_solve.log
  H2G_SOLVE_THREADS=$nt timeout 600 python scripts/solve_only.py 2 >> gpurun_out/r02n_solve.log 2>&1
done
H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 > gpurun_out/r02n_prof_levels.log 2>&1
H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 colored > gpurun_out/r02n_prof_levels_colored.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo "bench rc $?" >> gpurun_out/r02n_bench.err
timeout 1500 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02n_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02n_cfg3_1e-3.log
