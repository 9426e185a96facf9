#!/bin/bash
# ncu capture of one filter-degree kernel (stencil path or CSR) on one config.
#   scripts/prof_filter.sh <config> <st|csr> <kernel-regex> <out-name>
set -e
CFG=${1:-3}; PATH_=${2:-st}; KRE=${3:-stencil_kernel}; OUT=${4:-prof}
CMD="python scripts/bench_filter.py --configs $CFG --paths $PATH_ --reps 1"
$CMD > gpurun_out/${OUT}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 -o gpurun_out/$OUT $CMD > gpurun_out/${OUT}_ncu.log 2>&1
