#!/bin/bash
# Round-2 GPU session K: oracle rank noise on the config-4-geometry analog (eps 1e-2), full GPU tests.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out/golden
python - <<'PY' > gpurun_out/golden/save_h2_k.log 2>&1
import sys; sys.path.insert(0, ".")
import paper_1703_06155_b200 as h2g
from paper_1703_06155_b200.geometry import vie_grid_points
A = h2g.H2Matrix.build(vie_grid_points(32, 2.0), 64, 1.0, h2g.vie_kernel(32, 2.0), 1e-2)
A.save("/tmp/cfg4a_gpu.h2")
print("saved")
PY
timeout 1200 python scripts/oracle_rank_noise.py 4 gpurun_out/golden/cfg4a_rank_noise.json /tmp/cfg4a_gpu.h2 1e-2 > gpurun_out/golden/noise_k.log 2>&1; echo "noise rc $?" >> gpurun_out/golden/noise_k.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02k_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02k_pytest.log
