#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_gpu6.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu6.log
for lib in build/libarrabit_*.so; do
  echo "== $lib" >> gpurun_out/dmma.log
  ARRABIT_LIB=$PWD/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/dmma_bench.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/dmma_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['ms_per_step'], {k:round(v,2) for k,v in r['phase_ms_per_step'].items()}, 'gram TF', r['dense_gram']['achieved'])" >> gpurun_out/dmma.log
  ARRABIT_LIB=$PWD/$lib timeout 600 python scripts/profile_step.py --config 3 --reps 1 --warmup 1 --tiles 16 --band 10 2>&1 | grep "config" >> gpurun_out/dmma.log
done
echo done
