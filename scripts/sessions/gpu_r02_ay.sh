#!/bin/bash
# Round-2 GPU session AY (closing evidence of the final commit): full GPU tests, smoke, bench (both arms), ncu launch list of one factorize + solve.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=/tmp/h2g_ay; rm -rf $T; mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02ay_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02ay_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ay_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02ay_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02ay_bench_reference.json 2> gpurun_out/r02ay_bench_reference.err
timeout 900 python bench.py > gpurun_out/r02ay_bench.json 2> gpurun_out/r02ay_bench.err; echo "bench rc $?" >> gpurun_out/r02ay_bench.err
python scripts/profile_once.py 2 > gpurun_out/r02ay_plain.log 2>&1 || exit 1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches.csv python scripts/profile_once.py 2 > gpurun_out/r02ay_ncu_launch.log 2>&1
python scripts/launch_table.py $T/launches.csv > gpurun_out/r02ay_launch_table.txt 2>&1
python scripts/launch_summary.py $T/launches.csv >> gpurun_out/r02ay_launch_table.txt 2>&1
gzip -9 -c $T/launches.csv > gpurun_out/r02ay_launches.csv.gz
