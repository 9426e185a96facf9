#!/bin/bash
O=gpurun_out/gemmgrid
mkdir -p $O
python scripts/micro_gram_shapes.py > $O/shapes.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
echo done
