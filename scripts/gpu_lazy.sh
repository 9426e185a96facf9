#!/bin/bash
# lazy MPM normalisation: stencil/CSR tests + parity suite subset + A/B solve timing
O=gpurun_out/lazy
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_parity.py tests/test_gpu_parity_all.py tests/test_gpu_dist.py tests/test_gpu_colsplit.py -q -m gpu -k "not cfg5 and not cfg4" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for L in; do
  ARRABIT_LAZY_NORM=$L timeout 600 python scripts/rule_sweep.py --config 3 >> $O/ab.log 2>&1
  ARRABIT_LAZY_NORM=$L timeout 600 python scripts/rule_sweep.py --config 2 >> $O/ab.log 2>&1
done
echo done > $O/done
