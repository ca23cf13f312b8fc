#!/bin/bash
# Round-end measurement set: bench (C4 headline + C2 line), p sweep, launch list, ncu captures.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/re_bench_c4.json 2> gpurun_out/re_bench_c4.err
timeout 600 python bench.py --config C2 --no-cpu > gpurun_out/re_bench_c2.json 2> gpurun_out/re_bench_c2.err
timeout 600 python tools/p_sweep.py --out gpurun_out/re_p_sweep.json > gpurun_out/re_p_sweep.log 2>&1
bash tools/prof_all.sh > gpurun_out/re_prof_all.log 2>&1
tail -c 3000 gpurun_out/re_bench_c4.json gpurun_out/re_bench_c2.json
