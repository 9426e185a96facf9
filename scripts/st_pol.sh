#!/bin/bash
# L2 eviction policies of the stencil path (Y_j boxes / once-read operands / stores): 0 normal 1 last 2 first
for c in "1 2 2" "0 2 2" "0 0 0" "1 0 0" "0 2 0" "2 2 2"; do set -- $c
  echo "ypol=$1 spol=$2 opol=$3"
  ARRABIT_ST_YPOL=$1 ARRABIT_ST_SPOL=$2 ARRABIT_ST_OPOL=$3 python scripts/bench_filter.py --configs 3 --paths st --reps 3
done
