#!/bin/bash
# stencil path: one 1024-thread CTA per SM vs two 512-thread CTAs per SM
for t in 1024 512; do echo "threads=$t"; ARRABIT_ST_THREADS=$t ARRABIT_ST_VERBOSE=1 python scripts/bench_filter.py --configs 3 5 --paths st --reps 3 2>&1 | sort -u; done
