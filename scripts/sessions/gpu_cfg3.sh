mkdir -p gpurun_out
H2G_VERBOSE=2 timeout 1500 python scripts/try_config.py 3 > gpurun_out/cfg3.log 2>&1; echo "cfg3 exit $?" >> gpurun_out/cfg3.log
