#!/bin/bash
# Sweeps-rule tuning (R6): digits constant D and s_max on cfg1-4 (cfg4 at the
# reduced n = 4e5, k = 100 parity size).
O=gpurun_out/rule
mkdir -p $O
for cfg in "3" "2" "1" "4 --size 400000 --k 100"; do
  tag=$(echo $cfg | tr ' ' '_')
  ARRABIT_RANGE_DIGITS=8 timeout 600 python scripts/rule_sweep.py --config $cfg --save $O/ev_$tag.npy >> $O/sweep.log 2>&1
  for D in 10 12 14; do
    for S in 5 8; do
      ARRABIT_RANGE_DIGITS=$D timeout 600 python scripts/rule_sweep.py --config $cfg --smax $S --ref $O/ev_$tag.npy >> $O/sweep.log 2>&1
    done
  done
done
echo done >> $O/sweep.log
