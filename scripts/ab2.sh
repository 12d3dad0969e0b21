#!/bin/bash
mkdir -p gpurun_out
python scripts/membw.py > gpurun_out/membw.json 2>&1
for m in 1 2 3; do
  STG_FAST_CTAS_PER_SM=$m timeout 300 python bench.py --steps 8000 --no-cpu --no-extra > gpurun_out/bench_m$m.json 2>/dev/null
done
CMD="python scripts/prof_slab.py c4 3"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:persist -s 1 -c 2 \
    -o gpurun_out/prof_v2 $CMD > gpurun_out/ncu_v2.log 2>&1
