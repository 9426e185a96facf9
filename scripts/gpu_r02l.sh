#!/bin/bash
# round 2, session 6: stencil path on z-slabs (row partition) + regression of the single-GPU stencil path
mkdir -p gpurun_out/r02l
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_stencil.py -x -q -m gpu -rs > gpurun_out/r02l/pytest_dist_stencil.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02l/pytest_dist_stencil.log
tail -15 gpurun_out/r02l/pytest_dist_stencil.log
# cfg3 on 2 and 4 in-process ranks? (not a bench: correctness + per-rank kernel timing of a slab)
ARRABIT_ST_VERBOSE=1 timeout 600 python scripts/slab_filter_bench.py > gpurun_out/r02l/slab_filter_bench.log 2>&1
tail -20 gpurun_out/r02l/slab_filter_bench.log
