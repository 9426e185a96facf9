#!/bin/bash
# One GPU session (round 1, call 2): tests (incl. distributed on one GPU and full sizes),
# benches, per-config filter rates, ncu of the dominant filter-degree kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/pytest_dist.log 2>&1; echo "exit $?" >> gpurun_out/pytest_dist.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
for c in 3 4 5; do timeout 900 python scripts/profile_step.py --config $c --filter-only --reps 3 > gpurun_out/filter_cfg$c.log 2>&1; done
timeout 1200 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
PCMD="python scripts/profile_step.py --config 2 --filter-only"
timeout 600 $PCMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tile -s 25 -c 3 -o gpurun_out/prof_spmm2 $PCMD > gpurun_out/ncu_full.log 2>&1
echo done
