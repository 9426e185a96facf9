#!/bin/bash
set -x
mkdir -p gpurun_out
for lib in build/libarrabit_*.so; do
  echo "== $lib" >> gpurun_out/pf.log
  ARRABIT_LIB=$PWD/$lib W=220 timeout 300 python scripts/stream_test.py >> gpurun_out/pf.log 2>&1
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 2 --filter-only --reps 3 --tiles 32 64 2>&1 | grep "filter degree" >> gpurun_out/pf.log
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 3 --filter-only --reps 3 --tiles 16 --band 10 2>&1 | grep "filter degree" >> gpurun_out/pf.log
done
PCMD="python scripts/profile_step.py --config 3 --filter-only --reps 1 --warmup 1 --tiles 16 --band 10"
timeout 600 $PCMD > gpurun_out/plain_cfg3b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tile -s 5 -c 1 -o gpurun_out/prof_cfg3_band $PCMD > gpurun_out/ncu_cfg3b.log 2>&1
echo done
