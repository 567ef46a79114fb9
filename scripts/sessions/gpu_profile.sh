# Profiling pass on one B200: per-level table, ncu launch list, k_schur DRAM traffic, config-3 probe.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
H2G_VERBOSE=1 timeout 300 python scripts/prof_levels.py 2 > gpurun_out/prof_levels.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_once.py 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_schur --csv --log-file gpurun_out/schur_traffic.csv python scripts/profile_once.py 2 > gpurun_out/ncu_schur.log 2>&1
H2G_VERBOSE=2 timeout 900 python scripts/try_config.py 3 > gpurun_out/cfg3.log 2>&1; echo "cfg3 exit $?" >> gpurun_out/cfg3.log
