#!/bin/bash
# Round 1, call 5: filter kernel variants x tile sizes; y-band with small tiles; L2 micro-benchmark.
set -x
mkdir -p gpurun_out
./scripts/micro_l2 > gpurun_out/micro_l2.log 2>&1
for lib in build/libarrabit_*.so; do
  for c in 2 3; do
    echo "== $lib cfg$c" >> gpurun_out/variants2.log
    ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config $c --filter-only --reps 3 --tiles 16 32 64 2>&1 | grep "filter degree" >> gpurun_out/variants2.log
  done
done
timeout 900 python scripts/profile_step.py --config 3 --filter-only --reps 3 --tiles 8 16 32 --band 0 5 10 > gpurun_out/band2_cfg3.log 2>&1
timeout 1200 python scripts/profile_step.py --config 5 --filter-only --reps 2 --tiles 16 32 --band 0 4 8 > gpurun_out/band2_cfg5.log 2>&1
echo done
