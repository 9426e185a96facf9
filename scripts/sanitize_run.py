"""A short pass over every kernel family of the hot path for compute-sanitizer
(memcheck / racecheck / synccheck): cfg1 and cfg2 solves on the CSR kernels, a cfg2
solve and an interpolant-filter step on the stencil path (TMA + mbarrier pipeline), the
64x64 and 128x128 DMMA tiles, the residual pass, Gershgorin and the schedule check.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from synth import configs  # noqa: E402
import paper_1507_06078_b200 as arr  # noqa: E402


def main():
    for cid, grid in ((1, None), (2, None), (2, (300, 1, 300))):
        A, spec = configs.build_config(cid)
        ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
        if grid:
            ctx.eig_set_stencil(*grid)
        X = torch.from_numpy(configs.starting_block(spec)).cuda()
        ev, res, info = ctx.eig_solve(X, tol=1e-10, maxit=3)
        print(f"cfg{cid} grid={grid}: outer {info.outer} maxres {info.maxres:.2e} kernel {ctx.last_spmm_kernel}", flush=True)
        if grid:
            ctx.eig_set_filter("interp")
            ctx.eig_set_interval(info.a, info.b)
            ctx.filter_step(X, normalize=True)
        ctx.close()
    # 3-D 7-point and 27-point stencil paths on small grids, odd width, padded ld
    for A, grid in ((synth.laplacian_3d_potential(20, 2), (20, 20, 20)), (synth.stencil27_3d(14), (14, 14, 14))):
        ctx = arr.eig_init(arr.to_device_csr(A), 37, 1, 4, w=38)
        ctx.eig_set_stencil(*grid)
        buf = torch.randn(A.n, 40, dtype=torch.float64, device="cuda")
        X = buf[:, :38]
        ctx.eig_set_interval(0.0, 6.0)
        ctx.filter_step(X, normalize=True)
        Y = torch.zeros_like(X)
        ritz, rank = ctx.arr_project(X, Y)
        print(f"stencil n={A.n}: rank {rank} ritz0 {ritz[0]:.6f} kernel {ctx.last_spmm_kernel}", flush=True)
        ctx.close()
    # dense products at a large-tile shape
    n, w = 20000, 300
    ctx = arr.eig_init(arr.to_device_csr(synth.laplacian_1d(n)), w, 1, 2, w=w)
    Xg = torch.randn(n, w, dtype=torch.float64, device="cuda")
    G = torch.empty(w, w, dtype=torch.float64, device="cuda")
    ctx.gram(Xg, Xg, G)
    O = torch.empty_like(Xg)
    ctx.gemm(Xg, G, O)
    torch.cuda.synchronize()
    print("dense ok", flush=True)


if __name__ == "__main__":
    main()
