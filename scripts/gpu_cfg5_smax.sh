#!/bin/bash
# cfg5 (27-point 256^3, n = 16.8M, k = 256, d = 30, p = 2): the sweeps cap s_max (the D-rule
# allows > 5 sweeps per ARR here: |T_30| amplifies ~2.4x per sweep)
O=gpurun_out/cfg5smax
mkdir -p $O
for S in 5 10 20; do
  timeout 1500 python scripts/rule_sweep.py --config 5 --smax $S --reps 1 >> $O/sweep.log 2>&1
done
echo done >> $O/sweep.log
