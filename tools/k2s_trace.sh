#!/bin/bash
# K2s per-step clock64 trace (leaf 0) at several p: HPS_K2S_TRACE=1 through tools/p_sweep.py.
for p in ${@:-8 10 12}; do
  HPS_K2S_TRACE=1 timeout 120 python tools/p_sweep.py --ps $p --reps 1 2>&1 | grep -E "k2s trace|\"p\"" | cut -c1-600
done
