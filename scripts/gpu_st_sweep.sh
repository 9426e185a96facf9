#!/bin/bash
# Stencil-path filter degree: static vs ticket-ordered work items, z-chunks, plus-shaped boxes.
O=gpurun_out/st_sweep
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stencil.py -q -x > $O/pytest_stencil.log 2>&1; echo "exit $?" >> $O/pytest_stencil.log
run() { tag=$1; shift; echo "== $tag" >> $O/sweep.log; env "$@" ARRABIT_ST_VERBOSE=1 timeout 600 python scripts/bench_filter.py --configs $CFG --paths st --reps 3 >> $O/sweep.log 2>&1; }
CFG=3
run "cfg3 static whole-lines" ARRABIT_ST_DYN=0 ARRABIT_ST_PLUS=0
run "cfg3 dyn nzc1 whole" ARRABIT_ST_DYN=1 ARRABIT_ST_PLUS=0 ARRABIT_ST_NZC=1
run "cfg3 dyn nzc1 plus" ARRABIT_ST_DYN=1 ARRABIT_ST_PLUS=1 ARRABIT_ST_NZC=1
run "cfg3 dyn nzc2 plus" ARRABIT_ST_DYN=1 ARRABIT_ST_PLUS=1 ARRABIT_ST_NZC=2
run "cfg3 dyn nzc4 plus" ARRABIT_ST_DYN=1 ARRABIT_ST_PLUS=1 ARRABIT_ST_NZC=4
run "cfg3 static plus" ARRABIT_ST_DYN=0 ARRABIT_ST_PLUS=1
CFG=5
run "cfg5 static" ARRABIT_ST_DYN=0
run "cfg5 dyn nzc1" ARRABIT_ST_DYN=1 ARRABIT_ST_NZC=1
run "cfg5 dyn nzc4" ARRABIT_ST_DYN=1 ARRABIT_ST_NZC=4
echo done >> $O/sweep.log
