#!/bin/bash
# Round-2 GPU session AQ (closing evidence of the committed state): full GPU tests, smoke, bench (both arms), ncu --set full of the grouped 64-RHS dataflow solve kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=/tmp/h2g_aq; rm -rf $T; mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02aq_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02aq_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aq_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02aq_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02aq_bench_reference.json 2> gpurun_out/r02aq_bench_reference.err
timeout 900 python bench.py > gpurun_out/r02aq_bench.json 2> gpurun_out/r02aq_bench.err; echo "bench rc $?" >> gpurun_out/r02aq_bench.err
timeout 600 python scripts/solve_only.py 2 > gpurun_out/r02aq_solve_plain.log 2>&1 || exit 1
timeout 1200 $NCU --set full --clock-control none -k regex:flow --launch-skip 72 --launch-count 12 -o $T/flow64 -f python scripts/solve_only.py 2 > gpurun_out/r02aq_ncu_flow64.log 2>&1
$NCU -i $T/flow64.ncu-rep --page raw --csv > gpurun_out/r02aq_flow64.raw.csv 2>/dev/null
python scripts/ncu_raw_summary.py gpurun_out/r02aq_flow64.raw.csv > gpurun_out/r02aq_flow64_summary.txt 2>&1
du -sh gpurun_out
