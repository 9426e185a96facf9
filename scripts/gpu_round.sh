#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
for lib in build/libarrabit_*.so; do
  echo "== $lib" >> gpurun_out/ws2.log
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 2 --filter-only --reps 3 --tiles 16 32 64 2>&1 | grep "filter degree" >> gpurun_out/ws2.log
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 3 --filter-only --reps 3 --tiles 16 32 --band 0 10 2>&1 | grep "filter degree" >> gpurun_out/ws2.log
done
timeout 900 python scripts/profile_step.py --config 5 --filter-only --reps 2 --tiles 32 --band 8 > gpurun_out/ws2_cfg5.log 2>&1
echo done
