#!/bin/bash
# Round-2 ncu captures (--set full, one launch each) of the dominant kernels.
set -x
mkdir -p gpurun_out
python tools/prof_k2.py --config C4 --n 296 > gpurun_out/p2_k2c4_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2_lu_schur -s 1 -c 1 \
    -o gpurun_out/p2_k2_c4 python tools/prof_k2.py --config C4 --n 296 > gpurun_out/p2_k2c4_ncu.log 2>&1
python tools/prof_k2.py --config C2 --n 592 > gpurun_out/p2_k2c2_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2_lu_lockstep -s 1 -c 1 \
    -o gpurun_out/p2_k2_c2 python tools/prof_k2.py --config C2 --n 592 > gpurun_out/p2_k2c2_ncu.log 2>&1
python tools/prof_k2.py --config C1 --n 256 > gpurun_out/p2_k2s_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2s_condense -s 1 -c 1 \
    -o gpurun_out/p2_k2s_c1 python tools/prof_k2.py --config C1 --n 256 > gpurun_out/p2_k2s_ncu.log 2>&1
python tools/prof_k4k5.py > gpurun_out/p2_k4_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k4_values -s 1 -c 1 \
    -o gpurun_out/p2_k4_c4 python tools/prof_k4k5.py > gpurun_out/p2_k4_ncu.log 2>&1
ls -la gpurun_out/p2_*.ncu-rep
