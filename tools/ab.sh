#!/bin/bash
# A/B timing of K2 on C4 (1184 leaves) and C2, fused (default) vs HPS_UNFUSED=1.
for mode in fused unfused; do
  if [ $mode = fused ]; then export HPS_FUSED=1; else unset HPS_FUSED; fi
  echo "== $mode"
  timeout 100 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
  timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
done
