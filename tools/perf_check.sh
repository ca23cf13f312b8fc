#!/bin/bash
# Parity + K2 timing for one code change: GPU parity tests, then K2 on C4/C2/C1.
set -o pipefail
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 100 python tools/prof_k2.py --config C4 --n 1184 --reps 2 2>&1 | tail -1
timeout 100 python tools/prof_k2.py --config C2 --n 2304 --reps 3 2>&1 | tail -1
timeout 100 python tools/prof_k2.py --config C1 --n 256 --reps 3 2>&1 | tail -1
