#!/bin/bash
# A/B of a dense-kernel change: shape micro-benchmarks, GPU parity, cfg2/cfg3 (and cfg4) solves.
O=gpurun_out/${AB_TAG:-dense_ab}
mkdir -p $O
ARRABIT_DMMA_BIG=0 python scripts/micro_gram_shapes.py > $O/shapes_big0.log 2>&1
python scripts/micro_gram_shapes.py > $O/shapes.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 1800 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
[ -n "$AB_CFG4" ] && timeout 1800 python bench.py --config 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_cfg4.json 2> $O/bench_cfg4.err
echo done
