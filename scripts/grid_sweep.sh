#!/bin/bash
# fast 3-D kernel: bench-loop time per R(U) vs the persistent grid size
# (0 = the default, occupancy x SMs = 444; 410 = ten equal rounds at c4)
mkdir -p gpurun_out
S=${1:-2000}
for g in 0 410 373 342 296 420 430; do
  for r in 1 2; do
    export STG_FAST_GRID=$g
    echo "grid=$g rep=$r $(python bench.py --steps $S --no-extra --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]*1e3,2), "us", round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])')"
  done
done > gpurun_out/grid_sweep_$S.log 2>&1
