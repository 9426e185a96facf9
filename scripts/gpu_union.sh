#!/bin/bash
# Union-staged SpMM: parity subset, then filter-degree timings with the plan on / off.
O=gpurun_out/union2
mkdir -p $O
export ARRABIT_UNION_VERBOSE=1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "filter or spmm or residual or solve_matches" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for U in 0 1; do
  for R in 64 128; do
    [ $U = 0 ] && [ $R != 64 ] && continue
    echo "== UNION=$U ROWS=$R" >> $O/filter.log
    ARRABIT_UNION=$U ARRABIT_UNION_ROWS=$R timeout 300 python scripts/profile_step.py --config 2 --filter-only --reps 3 >> $O/filter.log 2>&1
    ARRABIT_UNION=$U ARRABIT_UNION_ROWS=$R timeout 300 python scripts/profile_step.py --config 3 --filter-only --band 10 --tiles 16 --reps 3 >> $O/filter.log 2>&1
  done
done
for U in 0 1; do
  echo "== cfg5 UNION=$U" >> $O/filter.log
  ARRABIT_UNION=$U timeout 600 python scripts/profile_step.py --config 5 --filter-only --band -1 --reps 1 >> $O/filter.log 2>&1
done
echo done
