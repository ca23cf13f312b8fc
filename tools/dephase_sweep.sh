#!/bin/bash
for d in 0 300000 700000 1200000 2000000; do
  echo "dephase_ns=$d"
  HPS_DEPHASE_NS=$d timeout 300 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
done
for d in 0 100000 200000; do
  echo "C2 dephase_ns=$d"
  HPS_DEPHASE_NS=$d timeout 300 python tools/prof_k2.py --config C2 --n 2304 --reps 2 2>&1 | tail -1
done
