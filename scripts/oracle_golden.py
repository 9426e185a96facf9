"""Write oracle-only golden eigenvalues for the parity tests (calls only oracle/ and
synth/; no CUDA path).  SURVEY §8c-6: cfg3 by the oracle's orthonormalise-then-augment
ARR (the paper-literal pivoted QR of the n x 1650 Krylov block takes hours); cfg4 on
the same generator at n = 4e5, k = 100 (the full n = 4e6 solve needs ~100 GB).

    python scripts/oracle_golden.py --config 3 --arr cgs2 --eigh lapack
    python scripts/oracle_golden.py --config 4 --n 400000 --k 100 --arr qr
"""
import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from synth import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--n", type=int, default=None, help="generator size override (zipf: n; grids: edge)")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--arr", default="qr", choices=["qr", "cgs2"])
    ap.add_argument("--eigh", default="jacobi", choices=["jacobi", "lapack"],
                    help="the projected eigenproblem: the oracle's cyclic Jacobi, or LAPACK as a library step "
                         "(cfg3: m = 1650, Jacobi in numpy takes ~25 min per ARR)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    spec = configs.CONFIGS[args.config]
    tag = f"cfg{args.config}"
    if args.n or args.k:
        spec = dataclasses.replace(spec, size=args.n or spec.size, k=args.k or spec.k)
        tag += f"_n{spec.n}_k{spec.k}"
    A, spec = configs.build_config(spec)
    X0 = configs.starting_block(spec)
    import oracle.core as oc
    oc.EIGH = args.eigh
    t0 = time.time()
    r = oracle.solve(A, spec.k, spec.d, spec.p, X0, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max,
                     w=spec.w, arr_method=args.arr)
    out = {
        "source": "scripts/oracle_golden.py (oracle/ only)",
        "config": spec.name, "n": int(A.n), "nnz": int(A.nnz), "k": spec.k, "w": spec.w, "d": spec.d, "p": spec.p,
        "seed": spec.seed, "tol": spec.tol, "arr_method": args.arr, "eigh": args.eigh, "range_digits": float(oracle.RANGE_DIGITS),
        "converged": bool(r.converged), "outer": r.outer, "sweeps": r.sweeps,
        "max_residual": float(r.res.max()), "eigenvalues": [float(x) for x in r.mu],
        "residuals": [float(x) for x in r.res], "seconds": time.time() - t0,
        "log": r.log,
    }
    path = args.out or os.path.join(ROOT, "tests", "golden", f"oracle_{tag}_eigs.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("config", "converged", "outer", "sweeps", "max_residual", "seconds")}))


if __name__ == "__main__":
    main()
