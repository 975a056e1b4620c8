"""Measured fp64 GEMM throughput on this GPU (cuBLAS DGEMM via torch.matmul,
8192^3, best of 5, CUDA events): the denominator for the setup kernels'
DMMA efficiency (the hot path is HBM-bound and does not use it)."""
import json

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"fp64_gemm_tflops": 2 * n ** 3 / (best * 1e-3) / 1e12, "n": n, "ms": best,
                  "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM), best of 5"}))
