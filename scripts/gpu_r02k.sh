#!/bin/bash
# R23 test, smoke, and the cfg3 launch list of one bench step on the final tree
O=gpurun_out/r02k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_all.py -q -m gpu -k "cholqr_factor or principal or vs_oracle_solve" > $O/pytest_r23.log 2>&1; echo "pytest rc=$?" >> $O/pytest_r23.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv \
   python bench.py --steps 1 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
gzip -f $O/launches_cfg3.csv
echo done > $O/done
