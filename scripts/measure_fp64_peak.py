"""Measure the FP64 DGEMM peak on this GPU (cuBLAS via torch.matmul, 8192^3, 2 N^3 flops):
best of 10 (burst) and back-to-back for ~4 s (sustained).  The roofline denominator for the
DMMA sketch kernel is reported beside the MEASURED_PEAKS-derived figure."""
import json
import sys
import time

import torch

N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
c = torch.empty_like(a)
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch.matmul(a, b, out=c); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.time(); k = 0
e0.record()
while time.time() - t < 4.0:
    torch.matmul(a, b, out=c); k += 1
    if k % 8 == 0:
        torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sus = 2.0 * N ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"dgemm_fp64_tflops_burst": 2.0 * N ** 3 / best / 1e12, "dgemm_fp64_tflops_sustained": sus,
       "how": "torch.matmul fp64 8192^3 (cuBLAS), best of 10 / back-to-back ~4 s"}
print(json.dumps(out))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"))
