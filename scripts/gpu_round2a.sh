#!/bin/bash
# first full bench of the round-2 tree (cfg3 default), the 128x64 DMMA tile A/B, parity suite
python bench.py --steps 3 --warmup 2 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
echo "bench rc=$?"
ARRABIT_DMMA_TILE=1 python scripts/micro_gram_shapes.py --no-cublas > gpurun_out/dmma_tile1.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_all.py -q -x --durations=20 > gpurun_out/parity_all.log 2>&1
echo "parity rc=$?"
