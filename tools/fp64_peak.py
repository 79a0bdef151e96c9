"""Measured FP64 dense GEMM throughput (cuBLAS DGEMM via torch, DMMA) — the FP64 roofline denominator."""
import json, torch
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
for _ in range(2):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"fp64_dgemm_tflops": 2 * 8192 ** 3 / (best * 1e-3) / 1e12, "ms": best}))
