#!/bin/bash
# L2-prefetch distance of the stencil path (filter degree), then the DMMA tile A/B
for pf in 0 2 4 8; do echo "pf=$pf"; ARRABIT_ST_VERBOSE=1 ARRABIT_ST_PF=$pf python scripts/bench_filter.py --configs 3 --paths st --reps 3 2>&1 | grep -v "^$" | sort -u; done
for pf in 0 4; do echo "pf=$pf"; ARRABIT_ST_VERBOSE=1 ARRABIT_ST_PF=$pf python scripts/bench_filter.py --configs 5 --paths st --reps 2 2>&1 | sort -u; done
echo "== dmma big"; python scripts/micro_gram_shapes.py
echo "== dmma 64x64"; ARRABIT_DMMA_BIG=0 python scripts/micro_gram_shapes.py --no-cublas
