#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -x > gpurun_out/st_test.log 2>&1; echo "stencil tests rc=$?"
for v in 0 1; do echo "prev_ldg=$v"; ARRABIT_ST_PREVLDG=$v ARRABIT_ST_VERBOSE=1 python scripts/bench_filter.py --configs 3 --paths st --reps 3 2>&1 | sort -u; done > gpurun_out/prevldg.log
python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k "cfg4_solve or cfg3_solve" --durations=5 > gpurun_out/fullsize_solves.log 2>&1; echo "fullsize rc=$?"
