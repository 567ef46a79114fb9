#!/bin/bash
# Round-2 GPU session E (ncu only): the solve level kernels, k_schur at level 7
# of config 2, and the bench launch list.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python scripts/profile_once.py 2 > gpurun_out/r02e_plain.log 2>&1 && \
$NCU --set full --clock-control none --import-source on -k regex:k_fwd_level -c 2 -o gpurun_out/r02e_fwd python scripts/profile_once.py 2 > gpurun_out/r02e_ncu_fwd.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_bwd_level -s 4 -c 2 -o gpurun_out/r02e_bwd python scripts/profile_once.py 2 > gpurun_out/r02e_ncu_bwd.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_schur -s 2140 -c 2 -o gpurun_out/r02e_schur python scripts/profile_once.py 2 > gpurun_out/r02e_ncu_schur.log 2>&1
python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02e_bench_plain.json 2> gpurun_out/r02e_bench_plain.err && \
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02e_launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02e_ncu_launch.log 2>&1
ls -la gpurun_out/
