#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1500 python scripts/solve_progress.py --config 4 --maxit 16 > gpurun_out/progress3_cfg4.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg2_v5.json 2> gpurun_out/bench_cfg2_v5.err
bash scripts/gpu_round4.sh
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu5.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu5.log
echo done
