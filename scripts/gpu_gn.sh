#!/bin/bash
set -x
O=gpurun_out/gn2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "gn_inner or deflation or adaptive" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --adapt 4 --no-e2e --no-cpu-baseline > $O/bench_cfg2_adapt4.json 2> $O/bench_cfg2_adapt4.err
timeout 900 python bench.py --adapt 7 --no-e2e --no-cpu-baseline > $O/bench_cfg2_adapt7.json 2> $O/bench_cfg2_adapt7.err
timeout 1800 python bench.py --config 3 --adapt 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_adapt4.json 2> $O/bench_cfg3_adapt4.err
timeout 1800 python bench.py --config 3 --adapt 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_adapt3.json 2> $O/bench_cfg3_adapt3.err
echo done
