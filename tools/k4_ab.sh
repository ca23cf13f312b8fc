for v in k4m6 k4n1 k4n6 k4m6 k4n1 k4n6; do
  export HPS_LIB_PATH=$PWD/build/variants/$v.so
  echo "$v $(python tools/prof_k4k5.py 2>&1 | grep 'K4 rep 1')"
done
for v in k4n1 k4n6; do
  export HPS_LIB_PATH=$PWD/build/variants/$v.so
  echo "$v tests: $(python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -k 'reduced or multi or condense_assemble' 2>&1 | tail -1)"
done
