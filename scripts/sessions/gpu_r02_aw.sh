#!/bin/bash
# Round-2 GPU session AW (closing evidence of the committed state): full GPU tests, smoke, bench (both arms), ncu --set full of the 64-RHS solve launches, config 4 at eps 1e-4 with 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=/tmp/h2g_aw; rm -rf $T; mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02aw_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02aw_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02aw_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02aw_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02aw_bench_reference.json 2> gpurun_out/r02aw_bench_reference.err
timeout 900 python bench.py > gpurun_out/r02aw_bench.json 2> gpurun_out/r02aw_bench.err; echo "bench rc $?" >> gpurun_out/r02aw_bench.err
timeout 600 python scripts/solve_only.py 2 > gpurun_out/r02aw_solve_plain.log 2>&1
timeout 1200 $NCU --set full --clock-control none -k regex:flow --launch-skip 72 --launch-count 12 -o $T/flow64 -f python scripts/solve_only.py 2 > gpurun_out/r02aw_ncu_flow64.log 2>&1
$NCU -i $T/flow64.ncu-rep --page raw --csv > $T/flow64.raw.csv 2>/dev/null
python scripts/ncu_raw_summary.py $T/flow64.raw.csv > gpurun_out/r02aw_flow64_summary.txt 2>&1
timeout 1500 python scripts/try_config.py 4 reference 1e-4 64 > gpurun_out/r02aw_cfg4_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02aw_cfg4_1e-4.log
