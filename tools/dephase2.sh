#!/bin/bash
for d in 0 150000 400000 800000; do
  echo "dephase $d"
  HPS_DEPHASE_NS=$d timeout 100 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
  HPS_DEPHASE_NS=$d timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
done
