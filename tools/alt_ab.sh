#!/bin/bash
# A/B of SS_PASS_ALT (alternating basis-pass streaming direction) on small and large systems.
cd "$(dirname "$0")/.."
for c in c1 pipe3d c5_small; do
  for rep in 1 2; do
    for alt in 0 1; do
      CASE=$c TAG="$c alt=$alt" SS_PASS_ALT=$alt REPS=3 timeout 300 python tools/c1_public_ab.py
    done
  done
done
for c in c1 c2; do
  echo "== in-cycle $c (ms per k-bucket: base alt)"
  timeout 600 python tools/tick_compare.py '{"base": {}, "alt": {"SS_PASS_ALT": "1"}}' $c
done
for alt in 0 1; do
  SS_PASS_ALT=$alt SS_PROFILE_DUMP=/tmp/c5_alt$alt.csv timeout 600 python tools/profile_case.py c5 200 1 > /dev/null 2>&1
  python -c "import numpy as np; d=np.loadtxt('/tmp/c5_alt$alt.csv', delimiter=','); print('c5 alt=$alt spmv/A/B/C ms per cycle', d.sum(0).round(1))"
done
