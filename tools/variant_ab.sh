#!/bin/bash
# K2 A/B over library variants (build/variants/<name>.so, `make variant NAME=... ...`):
# min over reps of K2 device time at C4 (1184 leaves = 4 waves), C3 (1184), C2 (all 2304).
# Usage: tools/variant_ab.sh default name1 name2 ...
for v in "$@"; do
  if [ "$v" = default ]; then unset HPS_LIB_PATH; else export HPS_LIB_PATH=$PWD/build/variants/$v.so; fi
  for c in "C4 1184" "C3 1184" "C2 2304"; do
    set -- $c
    r=$(timeout 120 python tools/prof_k2.py --config $1 --n $2 --reps 3 2>&1 | grep "^rep" | awk '{print $7}' | sort -n | head -1)
    echo "$v $1 n=$2 K2_ms=$r"
  done
done
