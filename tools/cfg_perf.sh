#!/bin/bash
for cfg in 256 128; do
  export HPS_K2_CFG=$cfg
  echo "== HPS_K2_CFG=$cfg"
  timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
  timeout 100 python tools/prof_k2.py --config C1 --n 256 --reps 3 2>&1 | tail -1
done
unset HPS_K2_CFG
