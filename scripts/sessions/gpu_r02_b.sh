#!/bin/bash
# Round-2 GPU session B: tests (incl. config-2 parity), bench, segmented fill
# storage on configs 3 / 4.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02b_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc $?" >> gpurun_out/r02b_bench.err
timeout 1200 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02b_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02b_cfg4_1e-2.log
timeout 2400 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02b_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02b_cfg3_1e-4.log
