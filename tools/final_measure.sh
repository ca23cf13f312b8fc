#!/bin/bash
# Final measurement set of the round: full GPU test suite, bench lines C4/C3/C2/C1, p sweep,
# launch list of the headline bench command.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f_pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 600 python bench.py --config C3 --steps 10 --warmup 3 > gpurun_out/f_bench_c3.json 2> gpurun_out/f_bench_c3.err
timeout 600 python bench.py --config C2 --steps 20 --warmup 5 > gpurun_out/f_bench_c2.json 2> gpurun_out/f_bench_c2.err
timeout 600 python bench.py --config C1 --steps 20 --warmup 5 > gpurun_out/f_bench_c1.json 2> gpurun_out/f_bench_c1.err
timeout 900 python tools/p_sweep.py --out gpurun_out/f_p_sweep.json > gpurun_out/f_p_sweep.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-leaf-solve > gpurun_out/f_launches_c4.log 2>&1
tail -2 gpurun_out/f_pytest_gpu.log
for c in c4 c3 c2 c1; do tail -c 300 gpurun_out/f_bench_$c.json; echo; done
