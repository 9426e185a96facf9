"""Time one filter degree (the fused SpMM launches of filter_step) on a config, CSR
kernels vs the stencil path (eig_set_stencil), and report the algorithmic-byte rate.

    python scripts/bench_filter.py --configs 2 3 5 [--paths csr st] [--reps 3]
Bytes per degree: CSR 12 nnz + 8(n+1) + 24 n w (16 n w on the first
degree); the stencil path reads A as K diagonals: 8 K n + 24 n w.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from synth import configs  # noqa: E402
import paper_1507_06078_b200 as arr  # noqa: E402


def grid_of(spec):
    if spec.kind == "lap1d":
        return (spec.size, 1, 1)
    if spec.kind == "lap2d":
        return (spec.size, 1, spec.size)  # march along y
    return (spec.size, spec.size, spec.size)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 3, 5])
    ap.add_argument("--paths", nargs="+", default=["csr", "st"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--yband", action="store_true", help="CSR path with the y-band row order for 3-D grids")
    ap.add_argument("--ld-align", type=int, default=16, help="row stride of X rounded up to this many doubles")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for cid in args.configs:
        A, spec = configs.build_config(cid)
        w, d = spec.w, spec.d
        Ad = arr.to_device_csr(A)
        ldx = (w + args.ld_align - 1) // args.ld_align * args.ld_align
        X = torch.empty((A.n, ldx), dtype=torch.float64, device="cuda")[:, :w]
        for r0 in range(0, A.n, 1 << 21):
            r1 = min(A.n, r0 + (1 << 21))
            X[r0:r1] = torch.from_numpy(synth.gaussian_block_rows(A.n, w, spec.seed, r0, r1))
        X0 = torch.empty_like(X).copy_(X) if A.n * w * 8 < 40e9 else None
        rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
        upper = float(np.bincount(rows, weights=np.abs(A.val), minlength=A.n).max())
        del rows
        for path in args.paths:
            ctx = arr.eig_init(Ad, spec.k, 0, d, w=w)
            if path == "st":
                ctx.eig_set_stencil(*grid_of(spec))
            elif args.yband and spec.kind in ("lap3dV", "st27"):
                from paper_1507_06078_b200 import schedule
                by, tile = {"lap3dV": (10, 16), "st27": (8, 32)}[spec.kind]
                ctx.eig_set_schedule(*schedule.yband_3d(spec.size, spec.size, spec.size, by, tile))
            a = ctx.eig_gershgorin_lower()
            ctx.eig_set_interval(a, a + 0.9 * (upper - a))
            ctx.filter_step(X, normalize=True)
            torch.cuda.synchronize()
            ctx.eig_set_timing(True)
            for _ in range(args.reps):
                if X0 is not None:
                    X.copy_(X0)
                ctx.filter_step(X, normalize=True)
            ms, cnt = ctx.eig_phase_times()
            deg_ms = ms[0] / cnt[0]
            K = ctx.stencil_points
            ab = ctx.stencil_abytes if K else None
            amod = ab * A.n if K else 12 * A.nnz + 8 * (A.n + 1)
            byts = (amod + 16 * A.n * w + (d - 1) * (amod + 24 * A.n * w)) / d
            gbs = byts / (deg_ms / 1e3) / 1e9
            print(json.dumps({"config": spec.name, "path": path + ("+yband" if args.yband and path == "csr" else ""),
                              "w": w, "d": d, "K": K, "A_bytes_per_row": ab, "ms_per_degree": round(deg_ms, 4),
                              "bytes_per_degree": byts, "GBs": round(gbs, 1), "frac_of_measured": round(gbs / peak, 4)}),
                  flush=True)
            ctx.close()
        del X, X0, Ad
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
