"""Micro-timings of the small dense steps (torch -> cuSOLVER) and of our DMMA Gram/GEMM."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_1507_06078_b200 as arr

def t_ms(f, reps=10):
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps

for m in (200, 400, 500, 1000, 1500):
    a = torch.randn(m, m, dtype=torch.float64, device="cuda"); a = a @ a.T + m * torch.eye(m, dtype=torch.float64, device="cuda")
    print(f"m={m}: eigh {t_ms(lambda: torch.linalg.eigh(a)):.3f} ms  cholesky {t_ms(lambda: torch.linalg.cholesky(a)):.3f} ms  "
          f"inv_tri {t_ms(lambda: torch.linalg.solve_triangular(torch.linalg.cholesky(a), torch.eye(m, dtype=torch.float64, device='cuda'), upper=False)):.3f} ms")
A = synth.laplacian_1d(90000)
ctx = arr.eig_init(arr.to_device_csr(A), 200, 1, 1)
for (n, m1, m2) in [(90000, 200, 200), (90000, 400, 200), (1000000, 500, 500), (1000000, 1500, 500)]:
    if n != 90000:
        ctx = arr.eig_init(arr.to_device_csr(synth.laplacian_1d(n)), 500, 2, 1)
    X = torch.randn(n, m1, dtype=torch.float64, device="cuda"); Y = torch.randn(n, m2, dtype=torch.float64, device="cuda")
    G = torch.empty(m1, m2, dtype=torch.float64, device="cuda")
    B = torch.randn(m1, m2, dtype=torch.float64, device="cuda"); O = torch.empty(n, m2, dtype=torch.float64, device="cuda")
    tg = t_ms(lambda: ctx.gram(X, Y, G)); tm = t_ms(lambda: ctx.gemm(X, B, O))
    fl = 2 * n * m1 * m2 / 1e12
    tc = t_ms(lambda: torch.matmul(X.T, Y))
    print(f"n={n} m1={m1} m2={m2}: gram {tg:.3f} ms ({fl/tg*1e3:.1f} TF)  gemm {tm:.3f} ms ({fl/tm*1e3:.1f} TF)   cublas XtY {tc:.3f} ms ({fl/tc*1e3:.1f} TF)")
