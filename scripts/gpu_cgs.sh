#!/bin/bash
# block CGS passes of the augmentation (ARRABIT_CGS_PASSES=1: one pass, the sketch check then
# decides whether to re-project): solve time / outer / eigenvalue agreement on cfg1-4
O=gpurun_out/cgs
mkdir -p $O
for cfg in "3" "2" "4 --size 400000 --k 100" "1"; do
  tag=$(echo $cfg | tr ' ' '_')
  ARRABIT_CGS_PASSES=2 timeout 600 python scripts/rule_sweep.py --config $cfg --save $O/ev_$tag.npy >> $O/cgs.log 2>&1
  ARRABIT_CGS_PASSES=1 timeout 600 python scripts/rule_sweep.py --config $cfg --ref $O/ev_$tag.npy >> $O/cgs.log 2>&1
done
echo done >> $O/cgs.log
