#!/bin/bash
# Round-2 final evidence on the committed tree: full GPU suite, smoke, the default bench line
# (cfg3 + cfg2 secondary + e2e + cpu_baseline), the reference (oracle) arm, the launch list of
# one bench step, ncu --set full of the DMMA GEMM launches of one cfg3 ARR.
O=gpurun_out/final
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/bench_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg3.csv \
   python bench.py --steps 1 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 16 \
   -o $O/gemm3 python scripts/profile_step.py --config 3 --warmup 0 --reps 1 > $O/ncu_gemm3.log 2>&1
echo done > $O/done
