#!/bin/bash
# Round-2 GPU session H: full GPU tests, racecheck on a small case, config 4 at eps 1e-3 with 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02h_pytest.log
timeout 600 python scripts/sanitize_case.py > gpurun_out/r02h_plain.log 2>&1 && \
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 50 python scripts/sanitize_case.py > gpurun_out/r02h_racecheck.log 2>&1; echo "racecheck rc $?" >> gpurun_out/r02h_racecheck.log
timeout 2400 python scripts/try_config.py 4 reference 1e-3 64 > gpurun_out/r02h_cfg4_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02h_cfg4_1e-3.log
