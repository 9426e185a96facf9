#!/bin/bash
# Validation of the latest library (handle pool, stream-ordered allocations, H reuse) + split experiment.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu3.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu3.log
timeout 400 python scripts/profile_step.py --config 2 --filter-only --reps 3 --tiles 16 32 --split 1 2 > gpurun_out/split_cfg2.log 2>&1
timeout 600 python scripts/profile_step.py --config 3 --filter-only --reps 3 --tiles 16 --band 10 --split 1 2 > gpurun_out/split_cfg3.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg2_v3.json 2> gpurun_out/bench_cfg2_v3.err

timeout 1500 python scripts/solve_progress.py --config 4 --maxit 10 > gpurun_out/progress_cfg4.log 2>&1
echo done
