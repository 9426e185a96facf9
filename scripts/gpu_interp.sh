#!/bin/bash
set -x
mkdir -p gpurun_out/interp
O=gpurun_out/interp
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "interp or filter or spmm or solve_small or lean" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --filter interp --no-e2e --no-cpu-baseline > $O/bench_cfg2_interp.json 2> $O/bench_cfg2_interp.err
timeout 1800 python bench.py --config 3 --filter interp --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_interp.json 2> $O/bench_cfg3_interp.err
timeout 900 python bench.py --config 1 --no-e2e > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 900 python bench.py --config 1 --filter interp --no-e2e --no-cpu-baseline > $O/bench_cfg1_interp.json 2> $O/bench_cfg1_interp.err
echo done
