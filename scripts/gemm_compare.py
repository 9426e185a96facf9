"""ncu target: one cuBLAS DGEMM and one libarrabit DMMA GEMM of the ARR's Ritz / CGS shape
(X n x m1 times B m1 x 550, n = 1e6), three times each.

    ncu --set full -k regex:"gemm" python scripts/gemm_compare.py [m1]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_06078_b200 as arr  # noqa: E402
from scripts.micro_gram_shapes import Diag  # noqa: E402

m1 = int(sys.argv[1]) if len(sys.argv) > 1 else 1650
n, m2 = 1000000, 550
X = torch.randn(n, m1, dtype=torch.float64, device="cuda")
B = torch.randn(m1, m2, dtype=torch.float64, device="cuda")
O = torch.empty(n, m2, dtype=torch.float64, device="cuda")
ctx = arr.eig_init(arr.to_device_csr(Diag(n)), m1, 2, 2, w=m1)
for _ in range(3):
    torch.matmul(X, B, out=O)
    ctx.gemm(X, B, O)
torch.cuda.synchronize()
print("ok")
