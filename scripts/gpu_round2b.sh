#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_colsplit.py -q -x > gpurun_out/colsplit.log 2>&1; echo "colsplit rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity_all.py -q -x --durations=20 > gpurun_out/parity_all.log 2>&1; echo "parity rc=$?"
python scripts/prof_dense.py 1000000 550 > gpurun_out/prof_dense_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_kernel_ca|gemm_kernel_ca" -s 2 -c 2 -o gpurun_out/prof_dense_cfg3 python scripts/prof_dense.py 1000000 550 > gpurun_out/prof_dense_ncu.log 2>&1
echo "ncu rc=$?"
