#!/bin/bash
# Per-phase cycle split of K2 (HPS_PHASE_TIMERS) with a debug-knob build of the library:
#   make variant NAME=dbg EXTRA=-DHPS_DEBUG_KNOBS            (phase marks)
#   make variant NAME=dbgm EXTRA="-DHPS_DEBUG_KNOBS -DHPS_STRIP_MARKS"   (+ per-column marks)
# Usage: tools/phases.sh [variant]  (default dbg)
V=${1:-dbg}
export HPS_LIB_PATH=$PWD/build/variants/$V.so HPS_PHASE_TIMERS=1
timeout 100 python tools/prof_k2.py --config C4 --n 296 --reps 1 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C4 --n 148 --reps 1 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 1 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C2 --n 592 --reps 1 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C2 --n 148 --reps 1 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C3 --n 296 --reps 1 2>&1 | tail -3
