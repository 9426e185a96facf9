#!/bin/bash
# Time scripts/profile_step.py (filter only) with each tuning variant in build/.
# usage: tune_variants.sh "<profile_step args>" ["<args>" ...]
for lib in build/libarrabit_*.so; do
  for a in "$@"; do
    echo "== $lib $a"; ARRABIT_LIB=$PWD/$lib python scripts/profile_step.py $a --filter-only --reps 3 2>&1 | tail -1
  done
done
