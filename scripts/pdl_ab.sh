#!/bin/bash
# A/B: programmatic dependent launch on/off for the bench loop and the solves
mkdir -p gpurun_out
for r in 1 2; do
  for mode in pdl nopdl; do
    if [ $mode = nopdl ]; then export STG_NO_PDL=1; else unset STG_NO_PDL; fi
    echo "$mode bench $(python bench.py --steps 5000 --no-extra --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"]*1e3,2), "us", round(d["roofline"]["frac"],4), d["clocks"]["sm_mhz"])')"
    for c in c4 c2 c3; do echo "$mode $c $(python scripts/prof_solve.py $c 2>&1 | grep solve)"; done
  done
done > gpurun_out/pdl_ab.log 2>&1
