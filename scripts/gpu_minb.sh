#!/bin/bash
# GEMM kernel register budget (ARR_DMMA_MINB / stages build variants, build/): micro shapes
O=gpurun_out/minb
mkdir -p $O
timeout 600 python scripts/micro_gram_shapes.py --no-cublas 2>&1 | grep "gemm X B" > $O/default.log
for v in ARR_DMMA_MINB4 ARR_DMMA_MINB3_ARR_DMMA_STAGES3; do
  ARRABIT_LIB=build/libarrabit_$v.so timeout 600 python scripts/micro_gram_shapes.py --no-cublas 2>&1 | grep "gemm X B" > $O/$v.log
done
echo done > $O/done
