#!/bin/bash
# Row alignment of the blocks (ld multiple of 16 doubles vs 2) on the stencil filter; GPU
# parity tests after the change; ncu of the aligned stencil degree; DMMA tile variants.
O=gpurun_out/ld_sweep
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stencil.py tests/test_gpu_dist.py -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
run() { echo "== $1 | $2 | $3" >> $O/sweep.log; env $2 timeout 600 python scripts/bench_filter.py --paths st --reps 3 $3 >> $O/sweep.log 2>&1; }
run "cfg3 ld2"  "ARRABIT_ST_PLUS=0 ARRABIT_LD_ALIGN=2"  "--configs 3 --ld-align 2"
run "cfg3 ld16" "ARRABIT_ST_PLUS=0 ARRABIT_LD_ALIGN=16" "--configs 3 --ld-align 16"
run "cfg3 ld16 plus" "ARRABIT_ST_PLUS=1 ARRABIT_LD_ALIGN=16" "--configs 3 --ld-align 16"
run "cfg3 ld16 static" "ARRABIT_ST_PLUS=0 ARRABIT_LD_ALIGN=16 ARRABIT_ST_DYN=0" "--configs 3 --ld-align 16"
run "cfg5 ld2"  "ARRABIT_LD_ALIGN=2"  "--configs 5 --ld-align 2"
run "cfg5 ld16" "ARRABIT_LD_ALIGN=16" "--configs 5 --ld-align 16"
ARRABIT_ST_PLUS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel --launch-skip 4 -c 1 \
   -o $O/st3_ld16 python scripts/bench_filter.py --paths st --reps 1 --configs 3 --ld-align 16 > $O/ncu_st3.log 2>&1
bash scripts/gpu_dense_sweep.sh
echo done >> $O/sweep.log
