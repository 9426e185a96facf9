#!/bin/bash
# round 2, session 6: stencil path on z-slabs (row partition) + regression of the single-GPU stencil path
mkdir -p gpurun_out/r02l
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_stencil.py -x -q -m gpu -rs > gpurun_out/r02l/pytest_dist_stencil.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02l/pytest_dist_stencil.log
ARRABIT_SLAB_BND=stencil timeout 1500 python -m pytest tests/test_gpu_dist.py -x -q -m gpu -k stencil > gpurun_out/r02l/pytest_dist_stencil_ends.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02l/pytest_dist_stencil_ends.log
tail -5 gpurun_out/r02l/pytest_dist_stencil.log gpurun_out/r02l/pytest_dist_stencil_ends.log
# cfg3 slabs of G in-process ranks at full size: bitwise check + wall time of all ranks together
for m in csr stencil; do
  ARRABIT_SLAB_BND=$m timeout 600 python scripts/slab_filter_bench.py 3 > gpurun_out/r02l/slab_filter_bench_cfg3_$m.log 2>&1
  tail -4 gpurun_out/r02l/slab_filter_bench_cfg3_$m.log
done
