#!/bin/bash
# Per-column critical-path split of the pivot strips (thread 0 clock marks, marks build).
export HPS_LIB_PATH=$PWD/build/variants/marks.so HPS_PHASE_TIMERS=1
for c in 1 0; do
  echo "== ctas/SM cap $c"
  HPS_K2_CTAS=$c timeout 120 python tools/prof_k2.py --config C2 --n 2304 --reps 1 2>&1 | tail -3
  HPS_K2_CTAS=$c timeout 120 python tools/prof_k2.py --config C4 --n 296 --reps 1 2>&1 | tail -3
done
