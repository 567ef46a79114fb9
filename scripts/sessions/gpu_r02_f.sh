#!/bin/bash
# Round-2 GPU session F: tests (hooks, facade, interior-first parity), oracle
# rank self-noise with per-cluster ranks, config 3 at eps 1e-4, config 4 at
# eps 1e-4 with 64 RHS.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02f_pytest.log
python - <<'PY' > gpurun_out/golden/save_h2_f.log 2>&1
import sys; sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_grid_points
c = BASELINE_CONFIGS[2]
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.vie_kernel(c["cells"], c["side"]), c["eps"])
A.save("/tmp/cfg2_gpu.h2")
print("saved")
PY
timeout 1500 python scripts/oracle_rank_noise.py 2 gpurun_out/golden/cfg2_rank_noise.json /tmp/cfg2_gpu.h2 > gpurun_out/golden/noise_f.log 2>&1; echo "noise rc $?" >> gpurun_out/golden/noise_f.log
timeout 3000 python scripts/try_config.py 3 reference 1e-4 1 > gpurun_out/r02f_cfg3_1e-4.log 2>&1; echo "exit $?" >> gpurun_out/r02f_cfg3_1e-4.log
