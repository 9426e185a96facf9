"""Outer-iteration / sweep counts of the GPU solve over X0 seeds, with and without
guard vectors (w = k + q).  python scripts/iter_sensitivity.py [config] [q ...]"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth
from synth import configs
import paper_1507_06078_b200 as arr
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
qs = [int(q) for q in sys.argv[2:]] or [0, 20]
A, spec = configs.build_config(cid)
Ad = arr.to_device_csr(A)
for q in qs:
    w = spec.k + q
    ctx = arr.eig_init(Ad, spec.k, spec.p, spec.d, w=w)
    for seed in range(spec.seed, spec.seed + 5):
        X = torch.from_numpy(synth.gaussian_block(A.n, w, seed)).cuda()
        torch.cuda.synchronize(); t = time.perf_counter()
        ev, res, info = ctx.eig_solve(X, tol=spec.tol)
        torch.cuda.synchronize(); t = time.perf_counter() - t
        print(f"q={q} seed={seed}: conv={info.converged} outer={info.outer} sweeps={info.sweeps} maxres={info.maxres:.2e} "
              f"time={t*1e3:.1f} ms eigpairs/s={spec.k/t:.0f} sum={ev.sum():.12f}", flush=True)
