# Round-end evidence on one B200: GPU tests, bench line, ncu launch list and per-launch k_schur DRAM traffic
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_once.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_table.py gpurun_out/launches.csv > gpurun_out/launch_table.txt 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_schur --csv --log-file gpurun_out/schur_traffic.csv python scripts/profile_once.py 2 > gpurun_out/ncu_schur.log 2>&1
python scripts/schur_traffic.py gpurun_out/schur_traffic.csv 2 > gpurun_out/schur_traffic.json
timeout 900 $NCU --set full --import-source on --clock-control none -k regex:k_schur --launch-skip 2140 --launch-count 2 -o gpurun_out/schur_l7 -f python scripts/profile_once.py 2 > gpurun_out/ncu_full.log 2>&1
$NCU -i gpurun_out/schur_l7.ncu-rep --page raw --csv --metrics launch__grid_size,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/schur_l7_metrics.csv 2>&1
timeout 900 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_1e-2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
