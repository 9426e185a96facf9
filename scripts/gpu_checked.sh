#!/bin/bash
# the GPU suite's small / medium cases against the bounds-checked build (compute-sanitizer stand-in)
ARRABIT_LIB=$PWD/paper_1507_06078_b200/libarrabit_checked.so timeout 1500 python -m pytest -q -x \
  tests/test_gpu_stencil.py tests/test_gpu_parity.py tests/test_gpu_parity_all.py tests/test_gpu_dist.py \
  tests/test_gpu_colsplit.py tests/test_gpu_advice_fixes.py -k "not cfg5 and not cfg3 and not cfg4 and not full" \
  > gpurun_out/checked_build_tests.log 2>&1
echo "checked rc=$?"
python scripts/bench_filter.py --configs 3 --paths st --reps 2 > gpurun_out/prof_final_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 3 -c 1 -o gpurun_out/prof_st3_final \
  python scripts/bench_filter.py --configs 3 --paths st --reps 2 > gpurun_out/prof_final_ncu.log 2>&1
echo "ncu rc=$?"
