#!/bin/bash
TAG=$1; CFG=${2:-C4}; N=${3:-148}
python tools/prof_k2.py --config $CFG --n $N > gpurun_out/prof_${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_lu -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} python tools/prof_k2.py --config $CFG --n $N > gpurun_out/prof_${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof_${TAG}_ncu.log
