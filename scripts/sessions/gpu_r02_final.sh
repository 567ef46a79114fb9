#!/bin/bash
# Round-2 final evidence: full GPU tests, smoke, bench (both arms), ncu launch list, k_schur DRAM traffic, ncu --set full of the Schur tile and the dataflow solve kernels.
# Large intermediates stay in /tmp on the box; gpurun_out/ only receives summaries (64 MiB cap).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=/tmp/h2g_final; rm -rf $T; mkdir -p $T
NCU=/usr/local/cuda/bin/ncu
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02f_smoke.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench rc $?" >> gpurun_out/r02f_bench.err
python scripts/profile_once.py 2 > gpurun_out/r02f_plain.log 2>&1 || exit 1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches.csv python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_launch.log 2>&1
python scripts/launch_table.py $T/launches.csv > gpurun_out/r02f_launch_table.txt 2>&1
python scripts/launch_summary.py $T/launches.csv >> gpurun_out/r02f_launch_table.txt 2>&1
gzip -9 -c $T/launches.csv > gpurun_out/r02f_launches.csv.gz
timeout 1200 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_schur --csv --log-file $T/schur_traffic.csv python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_schur.log 2>&1
python scripts/schur_traffic.py $T/schur_traffic.csv 2 > gpurun_out/r02f_schur_traffic.json 2>&1
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_schur --launch-skip 2140 --launch-count 2 -o $T/schur_l7 -f python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_full_schur.log 2>&1
timeout 900 $NCU --set full --clock-control none -k regex:k_schur --launch-skip 1300 --launch-count 2 -o $T/schur_l9 -f python scripts/profile_once.py 2 >> gpurun_out/r02f_ncu_full_schur.log 2>&1
timeout 900 $NCU --set full --clock-control none -k regex:flow --launch-count 12 -o $T/flow -f python scripts/profile_once.py 2 > gpurun_out/r02f_ncu_full_flow.log 2>&1
for f in schur_l7 schur_l9 flow; do
  $NCU -i $T/$f.ncu-rep --page raw --csv > gpurun_out/r02f_$f.raw.csv 2>/dev/null
done
ls -la $T > gpurun_out/r02f_tmp_listing.txt
# the one report small enough to travel: the level-7 Schur launches with source
[ $(stat -c %s $T/schur_l7.ncu-rep) -lt 20000000 ] && cp $T/schur_l7.ncu-rep gpurun_out/r02f_schur_l7.ncu-rep
du -sh gpurun_out
