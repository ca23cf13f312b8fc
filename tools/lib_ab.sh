#!/bin/bash
# K2 timing + bitwise A/B of library builds against the first one:
#   tools/lib_ab.sh build/ab/base.so build/variants/x.so [...]   (CASES="C4 4736;C2 2304" to override)
CASES=${CASES:-"C4 4736;C3 1184;C2 2304"}
LIBS=("$@")
BASE=${LIBS[0]}
for lib in "${LIBS[@]}"; do
  HPS_LIB_PATH=$lib python tools/bitwise_ab.py /tmp/ab_$(basename $lib .so).npz > /dev/null 2>&1
  [ "$lib" != "$BASE" ] && echo "$(basename $lib .so) vs $(basename $BASE .so): $(python tools/bitwise_ab.py --cmp /tmp/ab_$(basename $BASE .so).npz /tmp/ab_$(basename $lib .so).npz)"
done
for rep in 1 2; do
  for lib in "${LIBS[@]}"; do
    IFS=';' read -ra CS <<< "$CASES"
    for c in "${CS[@]}"; do
      set -- $c
      r=$(HPS_LIB_PATH=$lib timeout 300 python tools/prof_k2.py --config $1 --n $2 --reps 3 2>&1 | grep "^rep" | awk '{print $7}' | sort -n | head -1)
      echo "$(basename $lib .so) $1 n=$2 K2_ms=$r"
    done
  done
done
