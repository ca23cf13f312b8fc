#!/bin/bash
python tools/prof_k4k5.py > gpurun_out/pb_k4k5_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k4_values|k5_backsolve" -c 2 -o gpurun_out/pb_k4k5 python tools/prof_k4k5.py > gpurun_out/pb_k4k5_ncu.log 2>&1
python tools/prof_k2.py --config C4 --n 296 > gpurun_out/pb_k1_plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:k1_assemble_kernel -s 1 -c 1 -o gpurun_out/pb_k1 python tools/prof_k2.py --config C4 --n 296 > gpurun_out/pb_k1_ncu.log 2>&1
