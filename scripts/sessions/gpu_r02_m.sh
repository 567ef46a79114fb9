#!/bin/bash
# Round-2 GPU session M (after the container restore): full GPU tests, bench line, config 3 at eps 1e-4, config 4 at eps 1e-2 with 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02m_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02m_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err; echo "bench rc $?" >> gpurun_out/r02m_bench.err
timeout 1800 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02m_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02m_cfg3_1e-4.log
timeout 1200 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02m_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02m_cfg4_1e-2.log
