#!/bin/bash
# D = 12 dynamic-range rule + per-kernel DMMA timing: full GPU suite, smoke, default bench,
# ncu --set full of the Gram kernels of one cfg3 ARR (traffic per launch).
O=gpurun_out/r02g
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_kernel -c 40 \
   -o $O/gram3 python scripts/profile_step.py --config 3 --warmup 0 --reps 1 > $O/ncu_gram3.log 2>&1
echo done > $O/done
