export HPS_LIB_PATH=$PWD/build/variants/dbg.so HPS_PHASE_TIMERS=1
for n in 296 1184 4736; do echo "== C4 n=$n"; timeout 200 python tools/prof_k2.py --config C4 --n $n --reps 1 2>&1 | tail -3; done
for n in 592 2304; do echo "== C2 n=$n"; timeout 100 python tools/prof_k2.py --config C2 --n $n --reps 1 2>&1 | tail -3; done
