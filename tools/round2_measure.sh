#!/bin/bash
# Measurement set: bench lines (C4 headline, C3, C2, C1), per-config DRAM traffic of the
# dominant kernel (ncu, one wave), launch list of the headline bench command.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/m_bench_c4.json 2> gpurun_out/m_bench_c4.err
timeout 600 python bench.py --config C3 > gpurun_out/m_bench_c3.json 2> gpurun_out/m_bench_c3.err
timeout 600 python bench.py --config C2 > gpurun_out/m_bench_c2.json 2> gpurun_out/m_bench_c2.err
timeout 600 python bench.py --config C1 > gpurun_out/m_bench_c1.json 2> gpurun_out/m_bench_c1.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for spec in "C4 296 42 k2_lu_schur_kernel" "C3 296 32 k2_lu_schur_kernel" "C2 592 22 k2_lu_lockstep_kernel" "C1 256 12 k2s_condense_kernel"; do
  set -- $spec
  python tools/prof_k2.py --config $1 --n $2 > /dev/null 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:"k2_lu|k2s_condense" -s 1 -c 1 --csv \
      --log-file gpurun_out/m_traffic_$1.csv python tools/prof_k2.py --config $1 --n $2 > /dev/null 2>&1
  python tools/k2_traffic.py gpurun_out/m_traffic_$1.csv $3 $2 $4 "ncu dram__bytes_read+write of one $2-leaf launch (tools/round2_measure.sh)"
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches_c4.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-leaf-solve > gpurun_out/m_launches_c4.log 2>&1
tail -c 600 gpurun_out/m_bench_c4.json gpurun_out/m_bench_c3.json gpurun_out/m_bench_c2.json gpurun_out/m_bench_c1.json
