#!/bin/bash
# Round-end profiling: launch list of the bench command, full captures of K2, K1, K4, K5.
set -x
BENCH="python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e"
$BENCH > gpurun_out/pa_bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pa_launches.csv $BENCH > gpurun_out/pa_launch_ncu.log 2>&1
python tools/prof_k2.py --config C4 --n 296 > gpurun_out/pa_k2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_lu_schur -s 1 -c 1 -o gpurun_out/pa_k2 python tools/prof_k2.py --config C4 --n 296 > gpurun_out/pa_k2_ncu.log 2>&1
ncu --set full --clock-control none -k regex:k1_assemble_kernel -s 1 -c 1 -o gpurun_out/pa_k1 python tools/prof_k2.py --config C4 --n 296 > gpurun_out/pa_k1_ncu.log 2>&1
python tools/prof_k4k5.py > gpurun_out/pa_k4k5_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k4_values|k5_backsolve" -c 2 -o gpurun_out/pa_k4k5 python tools/prof_k4k5.py > gpurun_out/pa_k4k5_ncu.log 2>&1
echo done
