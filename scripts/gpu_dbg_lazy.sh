#!/bin/bash
O=gpurun_out/dbg
mkdir -p $O
for L in 1 0; do
  echo "== LAZY=$L" >> $O/t.log
  ARRABIT_LAZY_NORM=$L timeout 300 python -m pytest tests/test_gpu_degenerate.py -q -m gpu -k repeated_top >> $O/t.log 2>&1
done
ARRABIT_LAZY_NORM=1 timeout 300 python - >> $O/t.log 2>&1 <<'PY'
import numpy as np, torch, synth
import paper_1507_06078_b200 as arr
n, k = 400, 5
d = np.linspace(1.0, 2.0, n); d[-3:] = 3.0
A = synth.generators.diagonal(d)
ctx = arr.eig_init(arr.to_device_csr(A), k, 1, 6, w=k + 2)
X0 = synth.gaussian_block(n, k + 2, 6)
try:
    ev, res, info = ctx.eig_solve(torch.from_numpy(X0).cuda(), tol=1e-10, maxit=40)
    print("ok", info.outer, info.sweeps)
except Exception as e:
    print("ERR", e)
for l in ctx.last_log: print({k: l[k] for k in ("outer", "s", "a", "b", "mu1", "maxres")})
PY
bash scripts/gpu_minb.sh
echo done > $O/done
