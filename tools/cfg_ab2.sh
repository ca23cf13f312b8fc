for v in dbg g128c5 g128c6; do
  export HPS_LIB_PATH=$PWD/build/variants/$v.so
  for ls in 0 1; do
    export HPS_LOCKSTEP=$ls
    r=$(timeout 120 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | grep "^rep" | awk '{print $7}' | sort -n | head -1)
    echo "$v LOCKSTEP=$ls C2 K2_ms=$r"
  done
done
