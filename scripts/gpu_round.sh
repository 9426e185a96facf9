#!/bin/bash
# Round 1, call 6: tests (small Cholesky kernel, L2 prefetch), variants, bench.
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
for lib in build/libarrabit_*.so; do
  echo "== $lib cfg2" >> gpurun_out/variants3.log
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 2 --filter-only --reps 3 --tiles 32 64 2>&1 | grep "filter degree" >> gpurun_out/variants3.log
  echo "== $lib cfg3" >> gpurun_out/variants3.log
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 3 --filter-only --reps 3 --tiles 16 32 --band 0 10 2>&1 | grep "filter degree" >> gpurun_out/variants3.log
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
