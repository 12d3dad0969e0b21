#!/bin/bash
# c4 / c3 solve time per STG_PDL_MASK (1 slab, 2 fdm, 4 vec, 8 precond)
mkdir -p gpurun_out
for r in 1 2; do
for m in 0 15 1 2 4 8 13 11 14; do
  echo "mask $m $(STG_PDL_MASK=$m python scripts/prof_solve.py c4 2>&1 | grep solve) | $(STG_PDL_MASK=$m python scripts/prof_solve.py c3 2>&1 | grep solve)"
done
done > gpurun_out/pdl_mask.log 2>&1
