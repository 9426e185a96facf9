#!/bin/bash
set -x
mkdir -p gpurun_out
for lib in build/libarrabit_*.so; do
  echo "== $lib" >> gpurun_out/dmma2.log
  ARRABIT_LIB=$PWD/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dmma_bench.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/dmma_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], {k:round(v,2) for k,v in r['phase_ms_per_step'].items()}, 'gram TF', r['dense_gram']['achieved'])" >> gpurun_out/dmma2.log
  ARRABIT_LIB=$PWD/$lib timeout 600 python scripts/profile_step.py --config 3 --reps 1 --warmup 1 --tiles 16 --band 10 2>&1 | grep "config" >> gpurun_out/dmma2.log
done
ARRABIT_LIB=$PWD/build/libarrabit_ARR_DMMA_STAGES3_ARR_DMMA_MINB4.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "gram or arr or solve_small" > gpurun_out/pytest_dmma.log 2>&1
echo done
