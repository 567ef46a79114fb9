#!/bin/bash
# Round-2 final evidence: full GPU tests, smoke, bench (both arms), ncu launch list, k_schur DRAM traffic, ncu --set full of the Schur tile and the dataflow solve kernels.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02f_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc $?" >> gpurun_out/r02f_bench.err
python scripts/profile_once.py 2 > gpurun_out/r02f_plain.log 2>&1 || exit 1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches.csv python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_launch.log 2>&1
python scripts/launch_table.py gpurun_out/r02f_launches.csv > gpurun_out/r02f_launch_table.txt 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_schur --csv --log-file gpurun_out/r02f_schur_traffic.csv python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_schur.log 2>&1
python scripts/schur_traffic.py gpurun_out/r02f_schur_traffic.csv 2 > gpurun_out/r02f_schur_traffic.json 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_schur --launch-skip 2140 --launch-count 2 -o gpurun_out/r02f_schur_l7 -f python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_full_schur.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_schur --launch-skip 1300 --launch-count 2 -o gpurun_out/r02f_schur_l9 -f python scripts/profile_once.py 2 >> gpurun_out/r02f_ncu_full_schur.log 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:flow --launch-count 12 -o gpurun_out/r02f_flow -f python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_full_flow.log 2>&1
for f in r02f_schur_l7 r02f_schur_l9 r02f_flow; do
  $NCU -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null
done
ls -la gpurun_out/ | head -40
