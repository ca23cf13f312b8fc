python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in default ${VARS:-notri}; do
  if [ $v = default ]; then unset HPS_LIB_PATH; else export HPS_LIB_PATH=$PWD/build/variants/$v.so; fi
  echo "== $v"
  HPS_PHASE_TIMERS=1 timeout 120 python tools/prof_k2.py --config C2 --n 2304 --reps 2 2>&1 | tail -2
  timeout 120 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
done
