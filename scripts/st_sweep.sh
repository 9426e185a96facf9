#!/bin/bash
# A/B of the stencil path's L2 promotion and work-item order (filter degree, cfg3 and cfg5)
for promo in 0 64 256; do for order in 0 1; do
  echo "promo=$promo order=$order"
  ARRABIT_ST_PROMO=$promo ARRABIT_ST_ORDER=$order python scripts/bench_filter.py --configs ${CFGS:-3 5} --paths st --reps 3
done; done
