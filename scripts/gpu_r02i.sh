#!/bin/bash
# A/B on one box: default Gram kernel vs the 8-granular sub-tile skipping build (ARR_DMMA_SKIP=1)
O=gpurun_out/r02i
mkdir -p $O
for r in 1 2; do
  echo "== default (rep $r)" >> $O/ab.log
  timeout 300 python scripts/micro_gram_shapes.py --no-cublas >> $O/ab.log 2>&1
  echo "== skip (rep $r)" >> $O/ab.log
  ARRABIT_LIB=$PWD/paper_1507_06078_b200/libarrabit_skip.so timeout 300 python scripts/micro_gram_shapes.py --no-cublas >> $O/ab.log 2>&1
done
echo done > $O/done
