#!/bin/bash
# A/B timing of two in-tree builds: tools/ab.sh "<grep pattern>" [reps]
pat="$1"; reps="${2:-2}"
for r in $(seq $reps); do for v in libmlb_a.so libmlb_b.so; do
  echo "$v $(MLB_LIB_VARIANT=$v python tools/ablate_spread.py 2>&1 | grep -E "$pat" | tr -s ' ' | tr '\n' ';')"
done; done
