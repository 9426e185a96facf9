#!/bin/bash
# Round 2 (session e) evidence on the committed stencil kernel: ncu --set full of one filter
# degree on cfg3 and cfg5 (traffic per launch), and the launch list of one cfg3 bench step.
O=gpurun_out/r02f
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 3 -c 1 \
   -o $O/st3 python scripts/bench_filter.py --configs 3 --paths st --reps 1 > $O/ncu_st3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 3 -c 1 \
   -o $O/st5 python scripts/bench_filter.py --configs 5 --paths st --reps 1 > $O/ncu_st5.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv \
   python bench.py --steps 1 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
echo done > $O/done
