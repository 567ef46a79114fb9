"""N>1 path on CPU: bench.py under torch.distributed.run with world_size 2
(gloo). The factorization does not shard (replicas only), so the
multi-rank contract is the reference arm's rank-0-only execution and the
replica driver's rendezvous/max-over-ranks reduction; both run here without a
GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_torchrun(args, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "bench.py")] + args
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)


def test_reference_arm_rank0_only_world2(monkeypatch):
    out = run_torchrun(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0"], 29611)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["value"] > 0 and rec["cpu_baseline"]["cores"] >= 1
    assert rec["cpu_baseline"]["nproc"] >= 1 and rec["cpu_baseline"]["cpu_model"]
    assert rec["config"]["n"] == 32768  # the GPU arm's workload (config 2); the sample is its octant


def test_max_over_ranks_reduction_gloo(tmp_path):
    """The replica driver's timing reduction (max over ranks) with gloo."""
    code = r'''
import os, torch, torch.distributed as dist
dist.init_process_group("gloo")
r = dist.get_rank()
t = torch.tensor([1.0 + r], dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
assert t.item() == 2.0
dist.barrier()
if r == 0: print("OK", t.item())
dist.destroy_process_group()
'''
    path = str(tmp_path / "_maxred.py")
    open(path, "w").write(code)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29612", path]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "OK 2.0" in out.stdout
