#!/bin/bash
for la in 1 0; do
  export HPS_LOOKAHEAD=$la
  echo "== HPS_LOOKAHEAD=$la"
  timeout 100 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
  timeout 100 python tools/prof_k2.py --config C4 --n 148 --reps 2 2>&1 | tail -1
  timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
  timeout 100 python tools/prof_k2.py --config C3 --n 1184 --reps 2 2>&1 | tail -1
done
