#!/bin/bash
set -x
O=gpurun_out/final4
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "adaptive" > $O/pytest_adapt.log 2>&1; echo "exit $?" >> $O/pytest_adapt.log
for lib in build/libarrabit_*.so; do
  echo "== $lib" >> $O/ws3.log
  ARRABIT_LIB=$PWD/$lib timeout 400 python scripts/profile_step.py --config 2 --filter-only --reps 5 --tiles 16 32 64 2>&1 | grep "filter degree" >> $O/ws3.log
done
echo done
