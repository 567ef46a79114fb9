#!/bin/bash
# Round-2 GPU session T: compact streamed chain (segments leave the device at their final size), staged-target Schur variant: tests, per-level Schur times with the variant on fine levels / everywhere / off, config 3 at eps 1e-3.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg2_parity.py tests/test_serialize.py -m gpu -q -x > gpurun_out/r02t_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02t_pytest.log
for pf in 128 0 1000; do
  echo "H2G_SCHUR_PF_BMAX=$pf" >> gpurun_out/r02t_prof.log
  H2G_SCHUR_PF_BMAX=$pf H2G_VERBOSE=1 timeout 600 python scripts/prof_levels.py 2 2>&1 | grep -E "schur|factor_ms" >> gpurun_out/r02t_prof.log
done
timeout 2400 python scripts/try_config.py 3 reference 1e-3 1 > gpurun_out/r02t_cfg3_1e-3.log 2>&1; echo "exit $?" >> gpurun_out/r02t_cfg3_1e-3.log
