#!/bin/bash
# ncu --set full of the final K2 at C4 (one 1,184-leaf launch: 4 leaves per persistent CTA,
# dynamic schedule) and of the lock-step K2 at C2; each command runs once without ncu first.
mkdir -p gpurun_out
python tools/prof_k2.py --config C4 --n 1184 > gpurun_out/pf_k2c4_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2_lu_schur -s 1 -c 1 \
    -o gpurun_out/pf_k2_c4 python tools/prof_k2.py --config C4 --n 1184 > gpurun_out/pf_k2c4_ncu.log 2>&1
python tools/prof_k2.py --config C2 --n 2304 > gpurun_out/pf_k2c2_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2_lu_lockstep -s 1 -c 1 \
    -o gpurun_out/pf_k2_c2 python tools/prof_k2.py --config C2 --n 2304 > gpurun_out/pf_k2c2_ncu.log 2>&1
ls -la gpurun_out/pf_*.ncu-rep
