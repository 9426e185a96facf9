"""Run the CPU ORACLE's full fixed-parameter solve on a config and record its
outer-iteration / sweep counts (used by bench.py to extrapolate the oracle's
eigenpairs/s from a bounded sample).  Calls only oracle/ and synth/.

    python scripts/oracle_reference_counts.py 2   ->  tests/golden/oracle_cfg2_counts.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import configs  # noqa: E402


def main(cid: int):
    A, spec = configs.build_config(cid)
    X0 = synth.starting_block(spec)
    t = time.time()
    r = oracle.solve(A, spec.k, spec.d, spec.p, X0, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max)
    out = dict(config=spec.name, converged=bool(r.converged), outer=r.outer, sweeps=r.sweeps,
               maxres=float(r.res.max()), eig_sum=float(r.mu.sum()), eig_top=float(r.mu[0]),
               eig_k=float(r.mu[-1]), seconds=time.time() - t, s_per_outer=[e["s"] for e in r.log],
               source="scripts/oracle_reference_counts.py (oracle only)")
    path = os.path.join(ROOT, "tests", "golden", f"oracle_cfg{cid}_counts.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
