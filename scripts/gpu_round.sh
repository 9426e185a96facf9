#!/bin/bash
# One GPU session: tests, smoke, bench, launch list + one full ncu capture of the filter kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1; free -g >> gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
BCMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 $BCMD > gpurun_out/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launch.log 2>&1
PCMD="python scripts/profile_step.py --config 2"
timeout 600 $PCMD > gpurun_out/plain_prof.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_tile -s 45 -c 3 -o gpurun_out/prof_spmm $PCMD > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -s 4 -c 2 -o gpurun_out/prof_gram $PCMD > gpurun_out/ncu_gram.log 2>&1
echo done
