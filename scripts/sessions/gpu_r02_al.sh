#!/bin/bash
# Round-2 GPU session AL: coloured / subtree orders against the reference-order oracle fixture on config 2.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cfg2_parity.py -m gpu -q > gpurun_out/r02al_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02al_pytest.log
