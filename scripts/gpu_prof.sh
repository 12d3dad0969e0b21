#!/bin/bash
# ncu evidence for the slab kernels (run only after the same command exits 0).
set -u
mkdir -p gpurun_out
CMD="python scripts/prof_slab.py ${PROF_CFG:-c4} 5"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:slab -s 2 -c 3 \
    -o gpurun_out/prof_slab $CMD > gpurun_out/ncu_full.log 2>&1
echo "exit $?" >> gpurun_out/ncu_full.log
