#!/bin/bash
# After the value-mode-1 alignment fix and the branch-free interior steps: stencil parity,
# filter rates on cfg2/3/5, ncu of cfg5.
O=gpurun_out/vmode2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stencil.py -q > $O/pytest_stencil.log 2>&1; echo "exit $?" >> $O/pytest_stencil.log
run() { echo "== $1 | $2 | $3" >> $O/sweep.log; env $2 timeout 600 python scripts/bench_filter.py --paths st --reps 3 $3 >> $O/sweep.log 2>&1; }
run "cfg3" "ARRABIT_ST_VERBOSE=1" "--configs 3"
run "cfg5" "ARRABIT_ST_VERBOSE=1" "--configs 5"
run "cfg2" "ARRABIT_ST_VERBOSE=1" "--configs 2 --paths st csr"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 4 -c 1 \
   -o $O/st5 python scripts/bench_filter.py --paths st --reps 1 --configs 5 > $O/ncu_st5.log 2>&1
echo done >> $O/sweep.log
