#!/bin/bash
# Round-2 GPU session L: oracle rank noise incl. the Gram-truncation variant on the config-2 input and the analog.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
python - <<'PY' > gpurun_out/golden/save_h2_l.log 2>&1
import sys; sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import BASELINE_CONFIGS, vie_grid_points
c = BASELINE_CONFIGS[2]
A = h2g.H2Matrix.build(vie_grid_points(c["cells"], c["side"]), c["leaf"], 1.0, h2g.vie_kernel(c["cells"], c["side"]), c["eps"])
A.save("/tmp/cfg2_gpu.h2")
B = h2g.H2Matrix.build(vie_grid_points(32, 2.0), 64, 1.0, h2g.vie_kernel(32, 2.0), 1e-2)
B.save("/tmp/cfg4a_gpu.h2")
print("saved")
PY
NOISE_GRAM=1 timeout 1200 python scripts/oracle_rank_noise.py 4 gpurun_out/golden/cfg4a_rank_noise.json /tmp/cfg4a_gpu.h2 1e-2 > gpurun_out/golden/noise_l4.log 2>&1; echo "noise rc $?" >> gpurun_out/golden/noise_l4.log
NOISE_GRAM=1 timeout 2400 python scripts/oracle_rank_noise.py 2 gpurun_out/golden/cfg2_rank_noise.json /tmp/cfg2_gpu.h2 > gpurun_out/golden/noise_l2.log 2>&1; echo "noise rc $?" >> gpurun_out/golden/noise_l2.log
