#!/bin/bash
# z-slab stencil path: value mode 0 (the K diagonals staged per plane) forced, both end-plane policies
O=gpurun_out/r02m
mkdir -p $O
for vm in 0 1; do for bnd in csr stencil; do
  ARRABIT_ST_VMODE=$vm ARRABIT_SLAB_BND=$bnd timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -m gpu -k stencil > $O/pytest_vm${vm}_${bnd}.log 2>&1
  echo "pytest rc=$? (ARRABIT_ST_VMODE=$vm ARRABIT_SLAB_BND=$bnd)" >> $O/pytest_vm${vm}_${bnd}.log
  tail -n 2 $O/pytest_vm${vm}_${bnd}.log
done; done
