#!/bin/bash
# H's block (p-1, p) from the CholeskyQR factor + symmetric diagonal block (R23):
# same-box A/B against the direct Gram (ARRABIT_H_RFACTOR=0) on cfg1-4, GPU suite, cfg3 bench
O=gpurun_out/r02j
mkdir -p $O
for cfg in "3" "2" "4 --size 400000 --k 100" "1"; do
  tag=$(echo $cfg | tr ' ' '_')
  ARRABIT_H_RFACTOR=0 timeout 600 python scripts/rule_sweep.py --config $cfg --save $O/ev_$tag.npy >> $O/ab.log 2>&1
  ARRABIT_H_RFACTOR=1 timeout 600 python scripts/rule_sweep.py --config $cfg --ref $O/ev_$tag.npy >> $O/ab.log 2>&1
done
timeout 2400 python -m pytest tests -x -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done > $O/done
