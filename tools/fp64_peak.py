"""Measured FP64 peaks on this B200, the denominators of the FP64 rooflines:
  * dense DGEMM (cuBLAS via torch, DMMA pipe) — Gram / normal blocks / Cholesky;
  * the FP64 FMA pipe (a register-resident DFMA chain kernel, 8 independent chains per thread,
    148·k CTAs) — the collocation assembly, whose work is FMAs plus a software tanh."""
import json
import torch
from torch.utils.cpp_extension import load_inline

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
out = {"fp64_dgemm_tflops": 2 * 8192 ** 3 / (best * 1e-3) / 1e12, "dgemm_ms": best}

src = r"""
#include <torch/extension.h>
__global__ void k_dfma(double* out, int iters, double s) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], s, 1e-9);
  }
  double acc = 0;
  for (int i = 0; i < 8; ++i) acc += x[i];
  if (acc == 12345.678) out[0] = acc;
}
void dfma(torch::Tensor out, int64_t blocks, int64_t iters) {
  k_dfma<<<blocks, 256>>>(out.data_ptr<double>(), (int)iters, 0.999999);
}
"""
mod = load_inline("rdd_fp64_peak", cpp_sources="void dfma(torch::Tensor out, int64_t blocks, int64_t iters);",
                  cuda_sources=src, functions=["dfma"],
                  extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
sms = torch.cuda.get_device_properties(0).multi_processor_count
o = torch.zeros(1, dtype=torch.float64, device="cuda")
blocks, iters = sms * 8, 20000
mod.dfma(o, blocks, 100)
torch.cuda.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); mod.dfma(o, blocks, iters); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
out["fp64_fma_tflops"] = 2.0 * blocks * 256 * 8 * iters / (best * 1e-3) / 1e12
out["dfma_ms"] = best
print(json.dumps(out))
