# one build -> measure iteration: GPU parity tests, bench line, eig1c phase timers
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
H2G_DEBUG=8 timeout 300 python scripts/time_factor.py 2 > gpurun_out/eigdbg.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_once.py 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/launch_table.py gpurun_out/launches.csv > gpurun_out/launch_table.txt 2>&1
