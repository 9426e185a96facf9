"""Diagnostic: the fixed-parameter outer loop of eig_solve (R3, R6, R10)
driven step by step through the C-ABI calls (filter_step / arr_project /
residuals) so the per-outer progress (sweeps s, interval b, max residual, time)
of a config can be watched.

    python scripts/solve_progress.py --config 4 --maxit 12
"""
import argparse
import math
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


def cheb(d, t):
    r0, r1 = 1.0, t
    for _ in range(1, d):
        r0, r1 = r1, 2 * t * r1 - r0
    return r1 if d else 1.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--maxit", type=int, default=12)
    ap.add_argument("--smax", type=int, default=5)
    args = ap.parse_args()
    A, spec = configs.build_config(args.config)
    w, k = spec.w, spec.k
    ctx = arr.eig_init(arr.to_device_csr(A), k, spec.p, spec.d, w=w)
    X = torch.empty((A.n, w), dtype=torch.float64, device="cuda")
    for r0 in range(0, A.n, 1 << 21):
        r1 = min(A.n, r0 + (1 << 21))
        blk = synth.gaussian_block_rows(A.n, k, spec.seed, r0, r1)
        if spec.q:
            blk = np.hstack([blk, synth.gaussian_block_rows(A.n, spec.q, spec.seed, r0, r1, stream=2)])
        X[r0:r1] = torch.from_numpy(blk)
    t0 = time.perf_counter()
    a = ctx.eig_gershgorin_lower()
    mu, _ = ctx.arr_project(X, None, p=0)
    b, mu1 = mu[w - 1], mu[0]
    if not a < b:
        a = b - 1e-8 * (abs(b) + 1)
    print(f"init: a={a:.6g} b={b:.6g} mu1={mu1:.6g} ({time.perf_counter() - t0:.1f} s)", flush=True)
    mono, prev = False, 0.0
    for outer in range(1, args.maxit + 1):
        ctx.eig_set_interval(a, b)
        c, e = (a + b) / 2, (b - a) / 2
        amp = abs(cheb(spec.d, (mu1 - c) / e))
        s = args.smax if amp <= 1 else (1 if not math.isfinite(amp) else int(min(max(math.floor(8 / math.log10(amp)), 1), args.smax)))
        t1 = time.perf_counter()
        for _ in range(s):
            ctx.filter_step(X, normalize=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        ritz, rank = ctx.arr_project(X, X)
        t3 = time.perf_counter()
        res = ctx.residuals(X[:, :k], ritz[:k])
        print(f"outer {outer}: s={s} amp={amp:.3g} b={b:.8g} rank={rank} maxres={res.max():.3e} "
              f"mu1={ritz[0]:.10g} mu_k={ritz[k - 1]:.10g}  filter {t2 - t1:.2f} s, arr {t3 - t2:.2f} s", flush=True)
        if res.max() <= spec.tol:
            break
        mono = mono or (outer > 1 and res.max() > 10 * prev)
        prev = res.max()
        bn = ritz[min(w, len(ritz) - 1)]
        b, mu1 = (max(b, bn) if mono else bn), ritz[0]
        if not a < b:
            a = b - 1e-8 * (abs(b) + 1)


if __name__ == "__main__":
    main()
