#!/bin/bash
# Stencil value modes (constant coefficients): parity + filter rates + ncu of cfg3 and cfg5.
O=gpurun_out/vmode
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stencil.py -q -x > $O/pytest_stencil.log 2>&1; echo "exit $?" >> $O/pytest_stencil.log
run() { echo "== $1 | $2 | $3" >> $O/sweep.log; env $2 timeout 600 python scripts/bench_filter.py --paths st --reps 3 $3 >> $O/sweep.log 2>&1; }
run "cfg3" "ARRABIT_ST_VERBOSE=1" "--configs 3"
run "cfg3 vmode0" "ARRABIT_ST_VMODE=0" "--configs 3"
run "cfg5" "ARRABIT_ST_VERBOSE=1" "--configs 5"
run "cfg2" "ARRABIT_ST_VERBOSE=1" "--configs 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 4 -c 1 \
   -o $O/st3 python scripts/bench_filter.py --paths st --reps 1 --configs 3 > $O/ncu_st3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:stencil_kernel --launch-skip 4 -c 1 \
   -o $O/st5 python scripts/bench_filter.py --paths st --reps 1 --configs 5 > $O/ncu_st5.log 2>&1
echo done >> $O/sweep.log
