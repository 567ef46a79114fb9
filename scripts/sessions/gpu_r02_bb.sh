#!/bin/bash
# Round-2 GPU session BB (closing evidence of the final commit): full GPU tests, smoke, bench (both arms).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02bb_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02bb_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bb_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02bb_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02bb_bench_reference.json 2> gpurun_out/r02bb_bench_reference.err
timeout 900 python bench.py > gpurun_out/r02bb_bench.json 2> gpurun_out/r02bb_bench.err; echo "bench rc $?" >> gpurun_out/r02bb_bench.err
