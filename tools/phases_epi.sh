#!/bin/bash
# Tile-job mainloop vs epilogue cycles (HPS_EPI_MARKS debug build):
#   make variant NAME=epi EXTRA="-DHPS_DEBUG_KNOBS -DHPS_EPI_MARKS"
export HPS_LIB_PATH=$PWD/build/variants/epi.so HPS_PHASE_TIMERS=1
timeout 200 python tools/prof_k2.py --config C4 --n 1184 --reps 1 2>&1 | tail -4
timeout 200 python tools/prof_k2.py --config C2 --n 2304 --reps 1 2>&1 | tail -4
