#!/bin/bash
# Software-pipelined DMMA variants vs the default 64x64 kernels; ncu of the Gram at the H shape.
O=gpurun_out/dense_pipe
mkdir -p $O
for v in 0 7 9 10 11; do
  ARRABIT_DMMA_TILE=$v timeout 300 python scripts/micro_gram_shapes.py --no-cublas > $O/var$v.log 2>&1
done
ARRABIT_DMMA_TILE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel --launch-skip 40 -c 1 \
   -o $O/gram0 python scripts/micro_gram_shapes.py --no-cublas > $O/ncu_gram0.log 2>&1
ARRABIT_DMMA_TILE=7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gram_kernel --launch-skip 40 -c 1 \
   -o $O/gram7 python scripts/micro_gram_shapes.py --no-cublas > $O/ncu_gram7.log 2>&1
echo done > $O/done
