#!/bin/bash
# Round 1 final validation of the committed tree: all GPU tests, smoke, the default bench
# line, the reference arm, and the ncu launch list of the same bench command.
set -x
O=gpurun_out/final9
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_launch.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
nvidia-smi -q -d CLOCK > $O/smi.txt 2>&1
echo done
