#!/bin/bash
# Round 1: the adaptive driver options measured (deflation/continuation, adaptive p/d).
set -x
O=gpurun_out/adapt
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "deflation or adaptive" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for a in 4 3 7; do
  timeout 900 python bench.py --adapt $a --no-e2e --no-cpu-baseline > $O/bench_cfg2_adapt$a.json 2> $O/bench_cfg2_adapt$a.err
done
timeout 1800 python bench.py --config 3 --adapt 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_adapt4.json 2> $O/bench_cfg3_adapt4.err
timeout 1800 python bench.py --config 3 --adapt 4 --filter interp --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3_adapt4_interp.json 2> $O/bench_cfg3_adapt4_interp.err
echo done
