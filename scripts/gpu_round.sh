#!/bin/bash
set -x
mkdir -p gpurun_out
./scripts/micro_eig > gpurun_out/micro_eig2.log 2>&1
for W in 220 64 512; do W=$W timeout 300 python scripts/stream_test.py >> gpurun_out/stream_test.log 2>&1; echo "-- W=$W" >> gpurun_out/stream_test.log; done
echo done
