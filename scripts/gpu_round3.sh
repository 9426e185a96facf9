#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/solve_progress.py --config 4 --maxit 20 > gpurun_out/progress2_cfg4.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu4.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu4.log
timeout 900 python bench.py > gpurun_out/bench_cfg2_v4.json 2> gpurun_out/bench_cfg2_v4.err
timeout 2400 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo done
