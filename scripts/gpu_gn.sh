#!/bin/bash
set -x
O=gpurun_out/gn
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gn_inner or deflation" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --inner-solver gn --no-e2e --no-cpu-baseline > $O/bench_cfg2_gn.json 2> $O/bench_cfg2_gn.err
timeout 1800 python bench.py --config 3 --inner-solver gn --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_gn.json 2> $O/bench_cfg3_gn.err
echo done
