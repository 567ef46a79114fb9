#!/bin/bash
# Round-2 GPU session J: Schur epilogue change (per-level rates, bench), analog parity at the config-4 geometry.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py -q -x > gpurun_out/r02j_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02j_pytest.log
H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 > gpurun_out/r02j_prof_levels.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc $?" >> gpurun_out/r02j_bench.err
timeout 600 python scripts/analog_parity.py tests/golden/cfg4a_eps1e-2 > gpurun_out/r02j_cfg4a_parity.log 2>&1
