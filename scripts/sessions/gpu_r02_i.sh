#!/bin/bash
# Round-2 GPU session I: per-level Schur rates at config 2, the config-4
# geometry at eps 1e-2 on a 32^3 analog (same h, leaf 64) against an oracle
# run on the box host, and the ncu launch list of one factorize + solve.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 > gpurun_out/r02i_prof_levels.log 2>&1
timeout 2400 python scripts/oracle_golden.py 4 gpurun_out/golden/cfg4a_eps1e-2 --h2 gpu --eps 1e-2 --cells 32 --side 2.0 > gpurun_out/golden/cfg4a_log.txt 2>&1; echo "golden rc $?" >> gpurun_out/golden/cfg4a_log.txt
timeout 600 python scripts/analog_parity.py gpurun_out/golden/cfg4a_eps1e-2 > gpurun_out/r02i_cfg4a_parity.log 2>&1
python scripts/profile_once.py 2 > gpurun_out/r02i_plain.log 2>&1 && \
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02i_launches.csv python scripts/profile_once.py 2 > gpurun_out/r02i_ncu_launch.log 2>&1; echo "ncu rc $?" >> gpurun_out/r02i_ncu_launch.log
ls -la gpurun_out/r02i_launches.csv
