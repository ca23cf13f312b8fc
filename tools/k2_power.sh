(for i in $(seq 1 60); do nvidia-smi -i 0 --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active,temperature.gpu --format=csv,noheader,nounits; sleep 0.5; done) > gpurun_out/pw.log 2>&1 &
SP=$!
python tools/prof_k2.py --config C4 --n 4736 --reps 4 > gpurun_out/pw_k2.log 2>&1
kill $SP 2>/dev/null
