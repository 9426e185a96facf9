#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_colsplit.py tests/test_gpu_advice_fixes.py -q -x > gpurun_out/colsplit.log 2>&1; echo "colsplit rc=$?"
timeout 1500 python -m pytest tests/test_gpu_parity_all.py -q -k "not cfg5" --durations=10 > gpurun_out/parity_all.log 2>&1; echo "parity rc=$?"
