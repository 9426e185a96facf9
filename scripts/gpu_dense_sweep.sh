#!/bin/bash
# DMMA Gram / GEMM tile-shape variants on the ARR shapes vs cuBLAS; cuBLAS kernel names.
O=gpurun_out/dense_sweep
mkdir -p $O
timeout 300 python scripts/micro_gram_shapes.py --cublas-only > $O/cublas.log 2>&1
for v in 0 1 2 3 4 5 6; do
  ARRABIT_DMMA_TILE=$v timeout 300 python scripts/micro_gram_shapes.py --no-cublas > $O/var$v.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,launch__shared_mem_per_block_dynamic,launch__occupancy_limit_registers,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --csv --log-file $O/cublas_kernels.csv python scripts/micro_gram_shapes.py --cublas-only > $O/ncu_cublas.log 2>&1
echo done > $O/done
