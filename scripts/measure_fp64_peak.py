"""Measures the FP64 roofline denominators on this B200 (MEASURED_PEAKS.json
has only bf16/HBM): cuBLAS DGEMM and ZGEMM 8192^3, best of N, CUDA events."""
import json
import sys

import torch


def bench(dtype, n=8192, reps=8):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    flops = (8 if dtype.is_complex else 2) * n ** 3
    return flops / best / 1e12


out = {"dgemm_tflops": bench(torch.float64), "zgemm_tflops": bench(torch.complex128, 4096), "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
