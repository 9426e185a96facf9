"""Reproduce the value-mode-1 stencil case (14^3 Laplacian + V, w = 98) in isolation."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1507_06078_b200 as arr
w = int(sys.argv[1]) if len(sys.argv) > 1 else 98
N = int(sys.argv[2]) if len(sys.argv) > 2 else 14
A = synth.laplacian_3d_potential(N, 2)
Ad = arr.to_device_csr(A)
c = arr.eig_init(Ad, k=w, p=0, d=5)
c.eig_set_stencil(N, N, N)
print("abytes", c.stencil_abytes, flush=True)
c.eig_set_interval(0.0, 9.0)
X = torch.from_numpy(synth.gaussian_block(A.n, w, 7)).cuda()
c.filter_step(X, normalize=False)
torch.cuda.synchronize()
print("ok", float(X.abs().max()), flush=True)
