#!/bin/bash
# Round-2 GPU session BE: the library rebuilt from clean (build()): smoke, parity tests, facade / CLI / serialization tests.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02be_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02be_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02be_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02be_pytest.log
