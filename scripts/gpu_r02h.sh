#!/bin/bash
# 8-granular DMMA sub-tile skipping (ragged w = 550 edges, upper-triangular B, symmetric
# diagonal): ARR shapes vs cuBLAS, dense parity tests, cfg3 bench
O=gpurun_out/r02h
mkdir -p $O
timeout 600 python scripts/micro_gram_shapes.py > $O/micro_gram_shapes.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_all.py tests/test_gpu_advice_fixes.py -x -q -m gpu > $O/pytest_dense.log 2>&1; echo "pytest rc=$?" >> $O/pytest_dense.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done > $O/done
