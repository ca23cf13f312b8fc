#!/bin/bash
# Per-phase cycle split of K2 (HPS_PHASE_TIMERS) for C4, C2 (both configs), C1.
export HPS_PHASE_TIMERS=1
timeout 100 python tools/prof_k2.py --config C4 --n 1184 --reps 1 2>&1 | tail -3
for cfg in 128 256; do
  HPS_K2_CFG=$cfg timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 1 2>&1 | tail -3
done
timeout 100 python tools/prof_k2.py --config C3 --n 1184 --reps 1 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C1 --n 256 --reps 1 2>&1 | tail -3
