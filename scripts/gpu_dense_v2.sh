#!/bin/bash
# DMMA tile variants 12-14 (8-warp CTAs) against the defaults (GEMM 0, Gram 7) and cuBLAS on
# the ARR shapes (scripts/micro_gram_shapes.py).
O=gpurun_out/dense_v2
mkdir -p $O
timeout 600 python scripts/micro_gram_shapes.py > $O/default.log 2>&1
for v in 12 13 14; do
  ARRABIT_DMMA_TILE=$v ARRABIT_DMMA_GRAM=$v timeout 600 python scripts/micro_gram_shapes.py --no-cublas > $O/v$v.log 2>&1
done
echo done > $O/done
