"""Tuning experiment for the dynamic-range sweeps rule (R6): one config's full
solve (stencil path on grids) with the digits constant D taken from ARRABIT_RANGE_DIGITS
and a given s_max; prints outer / sweeps / solve time / max residual and the leading
eigenvalues' spread against a reference run (--ref).

    ARRABIT_RANGE_DIGITS=12 python scripts/rule_sweep.py --config 3 --smax 5
"""
import argparse
import json
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
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--size", type=int, default=None)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--smax", type=int, default=5)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--inner", default="range")
    ap.add_argument("--save", default=None, help="write the eigenvalues here (.npy)")
    ap.add_argument("--ref", default=None, help="compare with these eigenvalues (.npy)")
    args = ap.parse_args()
    spec = configs.CONFIGS[args.config]
    if args.size or args.k:
        import dataclasses
        spec = dataclasses.replace(spec, size=args.size or spec.size, k=args.k or spec.k)
    A, spec = configs.build_config(spec)
    X0 = torch.from_numpy(configs.starting_block(spec))
    big = X0.numel() * 8 * (spec.p + 4) > 0.8 * torch.cuda.get_device_properties(0).total_memory
    X0d = X0.pin_memory() if big else X0.cuda()  # cfg5: X0 stays on the host (as in bench.py)
    X = torch.empty(X0.shape, dtype=torch.float64, device="cuda")  # before eig_init: a lean context if needed
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    grid = {"lap1d": (spec.size, 1, 1), "lap2d": (spec.size, 1, spec.size),
            "lap3dV": (spec.size,) * 3, "st27": (spec.size,) * 3}.get(spec.kind)
    if grid:
        ctx.eig_set_stencil(*grid)
    out = []
    for _ in range(args.reps):
        X.copy_(X0d)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev, res, info = ctx.eig_solve(X, tol=spec.tol, maxit=spec.maxit, s_max=args.smax, inner=args.inner)
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    r = {"config": spec.name, "env": {k: v for k, v in os.environ.items() if k.startswith("ARRABIT_")}, "smax": args.smax,
         "inner": args.inner, "converged": bool(info.converged), "outer": int(info.outer), "sweeps": int(info.sweeps),
         "maxres": float(res.max()), "solve_s": min(out), "s_per_outer": [int(l["s"]) for l in ctx.last_log]}
    if args.save:
        np.save(args.save, ev)
    if args.ref and os.path.exists(args.ref):
        e0 = np.load(args.ref)
        r["max_rel_diff_vs_ref"] = float(np.max(np.abs(ev - e0) / np.maximum(1.0, np.abs(e0))))
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
