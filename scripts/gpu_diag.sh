#!/bin/bash
O=gpurun_out/diag
mkdir -p $O
python paper_1507_06078_b200/build.py --checked > $O/build_checked.log 2>&1
for cfg in "98 14" "24 14" "98 16" "66 14" "40 14"; do
  echo "== $cfg" >> $O/log
  CUDA_LAUNCH_BLOCKING=1 ARRABIT_ST_VERBOSE=1 timeout 120 python scripts/diag_vmode1.py $cfg >> $O/log 2>&1
  echo "== checked $cfg" >> $O/log
  ARRABIT_LIB=paper_1507_06078_b200/libarrabit_checked.so CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/diag_vmode1.py $cfg >> $O/log 2>&1
done
echo done >> $O/log
