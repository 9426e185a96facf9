#!/bin/bash
# GEMM tile variants on the ARR shapes (Gram fixed at the default variant 7).
O=gpurun_out/dense_v3
mkdir -p $O
for v in 0 7 8 9 10 11 1 5 6; do
  ARRABIT_DMMA_TILE=$v ARRABIT_DMMA_GRAM=7 timeout 600 python scripts/micro_gram_shapes.py --no-cublas 2>&1 | grep "gemm X B" > $O/gemm_v$v.log
done
echo done > $O/done
