#!/bin/bash
# Round-2 final profiles (small outputs: gpurun copies back <= 64 MiB): the launch list of one
# bench step (gzipped) and ncu --set full of 4 DMMA GEMM launches of one cfg3 ARR.
O=gpurun_out/fprof
mkdir -p $O
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv \
   python bench.py --steps 1 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
gzip -f $O/launches_cfg3.csv
timeout 900 ncu --set full --clock-control none -k regex:gemm_kernel -c 4 \
   -o $O/gemm3 python scripts/profile_step.py --config 3 --warmup 0 --reps 1 > $O/ncu_gemm3.log 2>&1
ls -la $O > $O/ls.txt
echo done > $O/done
