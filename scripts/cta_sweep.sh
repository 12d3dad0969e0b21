#!/bin/bash
# fast 3-D kernel: bench-loop time per R(U) vs CTAs per SM
mkdir -p gpurun_out
for c in 2 3 4; do
  for r in 1 2; do
    echo "ctas=$c rep=$r $(STG_FAST_CTAS_PER_SM=$c python bench.py --steps 5000 --no-extra --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]*1e3,2), "us", round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])')"
  done
done > gpurun_out/cta_sweep.log 2>&1
