mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1500 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/cfg4_1e-2.log
timeout 1500 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/cfg3_1e-3.log
