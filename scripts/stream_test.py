"""Filter-degree rate vs sparsity structure at a fixed block (n = 90,000, w = 220):
diagonal (no gathers), 1-D tridiagonal (x-neighbours only), 2-D 5-point (cfg2).
Isolates the cost of the gathers from the streams (Y_{j-1} in, Y_{j+1} out)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1507_06078_b200 as arr  # noqa: E402

n, w, d = 90000, int(os.environ.get("W", "220")), 20
mats = {"diag": synth.diagonal(np.linspace(1.0, 2.0, n)), "tridiag": synth.laplacian_1d(n), "5pt": synth.laplacian_2d(300)}
X = torch.from_numpy(synth.gaussian_block(n, w, 1)).cuda()
for name, A in mats.items():
    ctx = arr.eig_init(arr.to_device_csr(A), w, 0, d)
    a = float(A.val.min()) - 4
    ctx.eig_set_interval(a, a + 8)
    for _ in range(2):
        ctx.filter_step(X, normalize=True)
    torch.cuda.synchronize()
    ctx.eig_set_timing(True)
    for _ in range(3):
        ctx.filter_step(X, normalize=True)
    ms, cnt = ctx.eig_phase_times()
    us = ms[0] / cnt[0] * 1e3
    bpl = (12 * A.nnz + 8 * (n + 1) + 16 * n * w + (d - 1) * (12 * A.nnz + 8 * (n + 1) + 24 * n * w)) / d
    print(f"{name:8s} nnz/row {A.nnz / n:4.1f}: {us:7.1f} us/degree  {bpl / us / 1e3:6.0f} GB/s algorithmic", flush=True)
    ctx.close()
