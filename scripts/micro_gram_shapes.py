"""cuBLAS (torch fp64 matmul) on the Gram / GEMM shapes of the cfg2/cfg3 solves, for
comparison with the hand-written DMMA kernels."""
import torch
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for n, w in [(90000, 220), (90000, 440), (1000000, 550), (1000000, 1100), (8192, 8192)]:
    X = torch.randn(n, w, dtype=torch.float64, device="cuda")
    if n == 8192:
        ms = t(lambda: X @ X); print(f"cuBLAS DGEMM {n}^3: {2*n**3/ms/1e9:.1f} TF/s"); continue
    ms = t(lambda: X.T @ X); print(f"cuBLAS X^T X n={n} w={w}: {ms*1e3:.0f} us {2*n*w*w/ms/1e9:.1f} TF/s")
    R = torch.randn(w, w, dtype=torch.float64, device="cuda")
    ms = t(lambda: X @ R); print(f"cuBLAS X R   n={n} w={w}: {ms*1e3:.0f} us {2*n*w*w/ms/1e9:.1f} TF/s")
    del X

# the library's own DMMA Gram / GEMM on the same shapes (through the C-ABI)
import numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_1507_06078_b200 as arr
class Diag:  # identity CSR of order n: the context only needs A.n for the dense products
    def __init__(self, n):
        self.n = n; self.row_ptr = np.arange(n + 1); self.col_idx = np.arange(n); self.val = np.ones(n)
for n, w in [(90000, 220), (90000, 440), (1000000, 550), (1000000, 1100)]:
    ctx = arr.eig_init(arr.to_device_csr(Diag(n)), w, 1, 2, w=w)
    X = torch.randn(n, w, dtype=torch.float64, device="cuda")
    G = torch.empty(w, w, dtype=torch.float64, device="cuda")
    ms = t(lambda: ctx.gram(X, X, G)); print(f"arr gram X^T X n={n} w={w}: {ms*1e3:.0f} us {2*n*w*w/ms/1e9:.1f} TF/s (alg flops)")
    Y = X.clone()
    ms = t(lambda: ctx.gram(X, Y, G)); print(f"arr gram X^T Y n={n} w={w}: {ms*1e3:.0f} us {2*n*w*w/ms/1e9:.1f} TF/s")
    R = torch.randn(w, w, dtype=torch.float64, device="cuda"); O = torch.empty_like(X)
    ms = t(lambda: ctx.gemm(X, R, O)); print(f"arr gemm X R   n={n} w={w}: {ms*1e3:.0f} us {2*n*w*w/ms/1e9:.1f} TF/s")
    ctx.close(); del X, Y, O
