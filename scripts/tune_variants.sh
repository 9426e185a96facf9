#!/bin/bash
# Time scripts/profile_step.py (filter only) with each tuning variant in build/.
for lib in build/libarrabit_*.so; do
  for cfg in "$@"; do
    echo "== $lib cfg=$cfg"; ARRABIT_LIB=$PWD/$lib python scripts/profile_step.py --config $cfg --filter-only --reps 3 2>&1 | tail -1
  done
done
