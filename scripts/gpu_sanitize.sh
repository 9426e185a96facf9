#!/bin/bash
# compute-sanitizer, ONE tool per gpurun call (B200_PROFILING.md): memcheck | racecheck | synccheck
TOOL=${1:-memcheck}
python scripts/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1 && \
compute-sanitizer --tool $TOOL --print-limit 50 python scripts/sanitize_run.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "rc=$?"
