"""One DMMA Gram (X^T Y) and one GEMM (X R) of the cfg3 ARR shapes, for an ncu capture."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1507_06078_b200 as arr
n, w = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000, int(sys.argv[2]) if len(sys.argv) > 2 else 550
class Diag:
    def __init__(self, n):
        self.n = n; self.row_ptr = np.arange(n + 1); self.col_idx = np.arange(n); self.val = np.ones(n)
ctx = arr.eig_init(arr.to_device_csr(Diag(n)), w, 1, 2, w=w)
X = torch.randn(n, w, dtype=torch.float64, device="cuda"); Y = X.clone()
G = torch.empty(w, w, dtype=torch.float64, device="cuda")
R = torch.randn(w, w, dtype=torch.float64, device="cuda"); O = torch.empty_like(X)
for _ in range(2):
    ctx.gram(X, Y, G); ctx.gemm(X, R, O)
torch.cuda.synchronize(); print("ok")
