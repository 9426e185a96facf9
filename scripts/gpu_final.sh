#!/bin/bash
# Round 1 final evidence: GPU tests, smoke, bench lines (cfg2 default + filters), launch list, ncu.
set -x
O=gpurun_out/final2
mkdir -p $O
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm,driver_version --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --config 1 --no-e2e > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --config 1 --filter interp --no-e2e --no-cpu-baseline > $O/bench_cfg1_interp.json 2> $O/bench_cfg1_interp.err
BCMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $BCMD > $O/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $BCMD > $O/ncu_launch.log 2>&1
PCMD="python scripts/profile_step.py --config 2 --filter-only --reps 1 --warmup 2"
timeout 300 $PCMD > $O/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_ws -s 25 -c 3 -o $O/prof_ws $PCMD > $O/ncu_full.log 2>&1
echo done
