"""Short driver for ncu: warm up, then run ONE filter_step (d degree launches),
ONE arr_project and ONE residuals pass of a config's hot path.

    python scripts/profile_step.py [--config 2] [--reps 1]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from synth import configs  # noqa: E402
import paper_1507_06078_b200 as arr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--k", type=int, default=None, help="override block width (filter only)")
    ap.add_argument("--filter-only", action="store_true")
    ap.add_argument("--size", type=int, default=None, help="override the generator size (grid edge or n)")
    ap.add_argument("--tiles", type=int, nargs="*", default=[0], help="ARRABIT_TILE values to try (0: default)")
    ap.add_argument("--split", type=int, nargs="*", default=[1], help="ARRABIT_SPLIT values to try")
    ap.add_argument("--band", type=int, nargs="*", default=[0],
                    help="3-D y-band schedule heights to try in turn (0 natural, -1 auto)")
    args = ap.parse_args()
    spec = configs.CONFIGS[args.config]
    if args.size:
        import dataclasses
        spec = dataclasses.replace(spec, size=args.size, name=f"{spec.name}@{args.size}")
    A, spec = configs.build_config(spec)
    k = args.k or spec.w
    Ad = arr.to_device_csr(A)
    X = torch.empty((A.n, k), dtype=torch.float64, device="cuda")
    for r0 in range(0, A.n, 1 << 21):  # seeded X0, uploaded in row chunks
        r1 = min(A.n, r0 + (1 << 21))
        X[r0:r1] = torch.from_numpy(synth.gaussian_block_rows(A.n, k, spec.seed, r0, r1))
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    upper = float(np.bincount(rows, weights=np.abs(A.val), minlength=A.n).max())
    Y = torch.empty_like(X) if not args.filter_only else None
    from paper_1507_06078_b200 import schedule
    import itertools
    ctx = None
    for tile, band, split in itertools.product(args.tiles, args.band, args.split):
      if tile:
          os.environ["ARRABIT_TILE"] = str(tile)
      os.environ["ARRABIT_SPLIT"] = str(split)
      if ctx is not None:
          ctx.close()
      ctx = arr.eig_init(Ad, k, spec.p if not args.filter_only else 0, spec.d)
      a = ctx.eig_gershgorin_lower()
      ctx.eig_set_interval(a, a + 0.9 * (upper - a))
      if True:
        if band and spec.kind in ("lap3dV", "st27"):
            N = spec.size
            by = schedule.auto_band(N, N, k) if band < 0 else band
            ctx.eig_set_schedule(*schedule.yband_3d(N, N, N, by, tile or 64))
            tag = f"tile={tile} split={split} y-band by={by}"
        else:
            ctx.eig_set_schedule(None)
            tag = f"tile={tile} split={split} natural order"
        for _ in range(args.warmup):
            ctx.filter_step(X, normalize=True)
            if not args.filter_only:
                ritz, _ = ctx.arr_project(X, Y)
                ctx.residuals(Y, ritz[:k])
        torch.cuda.synchronize()
        ctx.eig_set_timing(True)
        t = time.perf_counter()
        for _ in range(args.reps):
            ctx.filter_step(X, normalize=True)
            if not args.filter_only:
                ritz, _ = ctx.arr_project(X, Y)
                ctx.residuals(Y, ritz[:k])
        torch.cuda.synchronize()
        wall = time.perf_counter() - t
        ms, cnt = ctx.eig_phase_times()
        deg_us = ms[0] / max(cnt[0], 1) * 1e3
        bpl = (12 * A.nnz + 8 * (A.n + 1) + 16 * A.n * k + (spec.d - 1) * (12 * A.nnz + 8 * (A.n + 1) + 24 * A.n * k)) / spec.d
        print(f"[{tag}] filter degree: {bpl/1e6:.1f} MB algorithmic / {deg_us:.1f} us = {bpl/deg_us/1e3:.0f} GB/s")
        print(f"[{tag}] config {spec.name} k={k}: wall {wall*1e3:.2f} ms; filter {ms[0]:.3f} ms / {cnt[0]} degree launches "
              f"({deg_us:.1f} us each); arr {ms[1]:.3f} ms / {cnt[1]} [basis {ms[3]:.3f} H {ms[4]:.3f} "
              f"eig {ms[5]:.3f}]; residuals {ms[2]:.3f} ms / {cnt[2]}", flush=True)


if __name__ == "__main__":
    main()
