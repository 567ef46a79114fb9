#!/bin/bash
# Round-2 GPU session C: tests (serialize, CLI, parity), the oracle's rank
# self-noise on the GPU-built config-2 input, bench, fill segmentation cost,
# configs 3 / 4.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02c_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02c_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench rc $?" >> gpurun_out/r02c_bench.err
python - <<'PY' > gpurun_out/golden/save_h2.log 2>&1
import sys; sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_grid_points
c = BASELINE_CONFIGS[2]
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.vie_kernel(c["cells"], c["side"]), c["eps"])
A.save("/tmp/cfg2_gpu.h2")
print("saved")
PY
timeout 2400 python scripts/oracle_rank_noise.py 2 gpurun_out/golden/cfg2_rank_noise.json /tmp/cfg2_gpu.h2 > gpurun_out/golden/noise.log 2>&1; echo "noise rc $?" >> gpurun_out/golden/noise.log
H2G_FILL_SEGMENTS=16 timeout 600 python scripts/try_config.py 2 > gpurun_out/r02c_cfg2_seg16.log 2>&1
timeout 600 python scripts/try_config.py 2 > gpurun_out/r02c_cfg2_seg1.log 2>&1
timeout 1200 python scripts/try_config.py 4 reference 1e-2 64 > gpurun_out/r02c_cfg4_1e-2.log 2>&1; echo "exit $?" >> gpurun_out/r02c_cfg4_1e-2.log
timeout 2400 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02c_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02c_cfg3_1e-4.log
