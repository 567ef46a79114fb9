#!/bin/bash
# Round-2 GPU session G: dataflow solve (tests + bench), step-0 refinement vs rank parity at config 2.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_serialize.py tests/test_gpu_hooks.py tests/test_facade.py -q -x > gpurun_out/r02g_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r02g_pytest.log
timeout 600 python scripts/cfg2_rank_check.py > gpurun_out/r02g_rank_default.log 2>&1
H2G_DEBUG=4 timeout 600 python scripts/cfg2_rank_check.py > gpurun_out/r02g_rank_refine.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; echo "bench rc $?" >> gpurun_out/r02g_bench.err
H2G_SOLVE_BATCHED=1 timeout 300 python scripts/solve_only.py > gpurun_out/r02g_solve_batched.log 2>&1
timeout 300 python scripts/solve_only.py > gpurun_out/r02g_solve_flow.log 2>&1
