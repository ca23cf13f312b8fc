export HPS_LIB_PATH=$PWD/build/variants/dbg.so
for cfg in "0 -1" "256 1" "256 0" "128 0" "128 1"; do
  set -- $cfg
  export HPS_K2_CFG=$1 HPS_LOCKSTEP=$2
  for c in ${CFG_CASES:-"C2 2304" "C3 1184"}; do
    set -- $c
    r=$(timeout 120 python tools/prof_k2.py --config $1 --n $2 --reps 3 2>&1 | grep "^rep" | awk '{print $7}' | sort -n | head -1)
    echo "K2_CFG=$HPS_K2_CFG LOCKSTEP=$HPS_LOCKSTEP $1 n=$2 K2_ms=$r"
  done
done
