"""Measure the FP64 (DMMA) matmul peak of this B200 with cuBLAS DGEMM via torch
(8192^3, best of 10 = burst; back to back for 4 s = sustained), mirroring how
MEASURED_PEAKS.json measures bf16.  Writes profiles/peaks_fp64.json."""
import json
import os
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
burst = 2 * N ** 3 / best / 1e12
t0 = time.perf_counter(); n = 0
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 4.0:
    c = a @ b; n += 1
    if n % 8 == 0:
        torch.cuda.synchronize()
e1.record(); e1.synchronize()
sus = 2 * N ** 3 * n / (e0.elapsed_time(e1) / 1e3) / 1e12
# copy bandwidth check (same recipe as MEASURED_PEAKS hbm_gbs)
x = torch.empty(2 ** 30 // 8, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
bw = 0
for _ in range(10):
    e0.record(); y.copy_(x); e1.record(); e1.synchronize()
    bw = max(bw, 2 * x.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9)
out = {"fp64_dgemm_tflops_burst": burst, "fp64_dgemm_tflops_sustained": sus, "copy_gbs": bw,
       "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM): best of 10 (burst), back to back 4 s (sustained); "
              "copy of 1 GiB fp64 (read+write bytes), best of 10",
       "gpu": torch.cuda.get_device_name()}
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "peaks_fp64.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
