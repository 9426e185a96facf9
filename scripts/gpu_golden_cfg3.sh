#!/bin/bash
# The oracle's full cfg3 solve on the GPU box's host cores (oracle/ + synth/ only; the GPU is
# idle), then the GPU parity test against the file it wrote.  scripts/oracle_golden.py is the
# only writer of tests/golden/oracle_cfg3_eigs.json.
O=gpurun_out/golden
mkdir -p $O
nproc > $O/host.txt; lscpu | grep "Model name" >> $O/host.txt
ORACLE_VERBOSE=1 timeout 5400 python scripts/oracle_golden.py --config 3 --arr cgs2 --eigh lapack --out $O/oracle_cfg3_eigs.json > $O/golden_cfg3.log 2>&1
echo "golden rc=$?" >> $O/golden_cfg3.log
tail -n 8 $O/golden_cfg3.log
if [ -s $O/oracle_cfg3_eigs.json ]; then
  cp $O/oracle_cfg3_eigs.json tests/golden/oracle_cfg3_eigs.json
  timeout 900 python -m pytest tests/test_gpu_parity_all.py -x -q -m gpu -k "cfg3_vs_oracle" -rs > $O/pytest_cfg3_vs_oracle.log 2>&1
  echo "pytest rc=$?" >> $O/pytest_cfg3_vs_oracle.log
  tail -n 5 $O/pytest_cfg3_vs_oracle.log
fi
