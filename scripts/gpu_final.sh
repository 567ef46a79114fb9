# Round-end evidence on one B200: GPU tests, bench line, ncu launch list and per-launch k_schur DRAM traffic
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_once.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_table.py gpurun_out/launches.csv > gpurun_out/launch_table.txt 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_schur --csv --log-file gpurun_out/schur_traffic.csv python scripts/profile_once.py 2 > gpurun_out/ncu_schur.log 2>&1
python scripts/schur_traffic.py gpurun_out/schur_traffic.csv 2 > gpurun_out/schur_traffic.json
