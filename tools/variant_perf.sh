#!/bin/bash
# Time K2 for alternative builds of the library (build/libhps_<tag>.so swapped in).
cp paper_2211_14969_b200/_lib/libhps_leaf_b200.so /tmp/libhps_default.so
for lib in /tmp/libhps_default.so build/libhps_*.so; do
  cp $lib paper_2211_14969_b200/_lib/libhps_leaf_b200.so
  echo "== $lib"
  timeout 100 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
  timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
done
cp /tmp/libhps_default.so paper_2211_14969_b200/_lib/libhps_leaf_b200.so
