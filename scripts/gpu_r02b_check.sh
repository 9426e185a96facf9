#!/bin/bash
# Re-entry check of the restored tree: GPU tests, smoke, stencil plan + filter rates, bench line.
O=gpurun_out/r02b_check
mkdir -p $O
nvidia-smi -L > $O/smi.txt 2>&1
ARRABIT_ST_VERBOSE=1 timeout 600 python scripts/bench_filter.py --configs 3 --paths st --reps 3 > $O/filter_cfg3.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
echo done
