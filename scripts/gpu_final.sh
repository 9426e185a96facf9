#!/bin/bash
# Round 1: new-feature tests (smallest mode, exit rules, rcond rule) and the cfg3/cfg4 bench lines.
set -x
O=gpurun_out/final3
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "smallest or exit_rules or rcond or interp" > $O/pytest_new.log 2>&1; echo "exit $?" >> $O/pytest_new.log
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 1800 python bench.py --config 3 --filter interp --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_interp.json 2> $O/bench_cfg3_interp.err
timeout 2400 python bench.py --config 4 --steps 1 --warmup 1 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
echo done
