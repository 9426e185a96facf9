#!/bin/bash
# Round-2 final evidence on the committed tree: full GPU suite, smoke, the default bench line
# (cfg3 + cfg2 secondary + e2e + cpu_baseline), the reference (oracle) arm.
O=gpurun_out/final
mkdir -p $O
timeout 2400 python -m pytest tests -x -q -m gpu --durations=12 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/bench_reference.err
echo done > $O/done
