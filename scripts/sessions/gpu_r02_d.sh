#!/bin/bash
# Round-2 GPU session D: tests, bench, config 3 (eps 1e-4) with the staged
# merge, config 4 at eps 1e-4 with 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_cfg2_parity.py::test_ranks_within_oracle_noise > gpurun_out/r02d_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02d_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc $?" >> gpurun_out/r02d_bench.err
timeout 1200 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02d_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02d_cfg4_1e-2.log
timeout 2700 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02d_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02d_cfg3_1e-4.log
