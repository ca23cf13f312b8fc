#!/bin/bash
# K2 timing of library variants (build/variants/*.so) against the default build.
for v in default "$@"; do
  if [ $v = default ]; then unset HPS_LIB_PATH; else export HPS_LIB_PATH=$PWD/build/variants/$v.so; fi
  echo "== $v"
  timeout 120 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
  timeout 120 python tools/prof_k2.py --config C1 --n 256 --reps 3 2>&1 | tail -1
done
