#!/bin/bash
# Phase split with 1 vs default co-resident K2 CTAs per SM (FP64 pipe contention probe).
export HPS_PHASE_TIMERS=1
for c in 1 0; do
  echo "== HPS_K2_CTAS=$c"
  HPS_K2_CTAS=$c timeout 100 python tools/prof_k2.py --config C4 --n 296 --reps 2 2>&1 | tail -2
  HPS_K2_CTAS=$c timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 2 2>&1 | tail -2
done
