#!/bin/bash
O=gpurun_out/gemm_ncu
mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:"gemm|nvjet|xmma|cutlass" -c 6 -o $O/gemm1650 python scripts/gemm_compare.py 1650 > $O/ncu.log 2>&1
echo done > $O/done
