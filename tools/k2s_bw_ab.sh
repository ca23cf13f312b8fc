#!/bin/bash
# K2s block-width A/B: default lib (K2S_BW=4) vs build/variants/bw{1,2}.so, HPS_SMALL=1.
for p in ${@:-6 7 8 9 10 11 12}; do
  line="p=$p"
  for lib in default build/variants/bw2.so build/variants/bw1.so; do
    if [ "$lib" = default ]; then unset HPS_LIB_PATH; else export HPS_LIB_PATH=$PWD/$lib; fi
    ms=$(HPS_SMALL=1 timeout 100 python tools/p_sweep.py --ps $p --reps 2 2>/dev/null | python -c "import json,sys; print('%.3f' % json.loads(sys.stdin.read())['ms_slice'])")
    line="$line  $(basename $lib):$ms"
  done
  echo "$line"
done
