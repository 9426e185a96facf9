#!/bin/bash
# Round 1: bench lines (cfg2 default + cfg3/4/5), launch list and ncu capture of the dominant kernel.
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
BCMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $BCMD > gpurun_out/ncu_launch2.log 2>&1
PCMD="python scripts/profile_step.py --config 2 --filter-only --reps 1 --warmup 2"
timeout 300 $PCMD > gpurun_out/plain_prof2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_ws -s 25 -c 3 -o gpurun_out/prof_ws_cfg2 $PCMD > gpurun_out/ncu_ws.log 2>&1
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 2400 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 2400 python bench.py --config 5 --steps 1 --warmup 1 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo done
