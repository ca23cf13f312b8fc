#!/bin/bash
# K2 timing + bitwise A/B of two library builds: tools/lib_ab.sh build/ab/base.so build/ab/new.so
A=$1; B=$2
for lib in $A $B; do
  HPS_LIB_PATH=$lib python tools/bitwise_ab.py gpurun_out/ab_$(basename $lib .so).npz
done
python tools/bitwise_ab.py --cmp gpurun_out/ab_$(basename $A .so).npz gpurun_out/ab_$(basename $B .so).npz
for rep in 1 2; do
for lib in $A $B; do
  for c in "C4 4736" "C3 1184" "C2 2304"; do
    set -- $c
    r=$(HPS_LIB_PATH=$lib timeout 300 python tools/prof_k2.py --config $1 --n $2 --reps 3 2>&1 | grep "^rep" | awk '{print $7}' | sort -n | head -1)
    echo "$(basename $lib .so) $1 n=$2 K2_ms=$r"
  done
done
done
