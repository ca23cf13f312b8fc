#!/bin/bash
# Parity, timing and one ncu capture of K2 for C4 and C2 with the current code.
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C4 C2; do
  n=296; [ $c = C2 ] && n=2304
  timeout 120 python tools/prof_k2.py --config $c --n $n --reps 3 2>&1 | tail -1
done
bash tools/prof_run.sh cur_c4 C4 296
bash tools/prof_run.sh cur_c2 C2 2304
