#!/bin/bash
# Round-2 (second session) evidence on the GPU box: --set full captures of the
# new kernels inside warm solves (fused fdm3 + couplings and the plain block
# apply in a c4 solve, k_offdiag in a c2 solve, the sweep kernels in a c3
# solve) and of the headline R(U) kernel, then their markdown summary.
set -u
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/ev2; mkdir -p $O
F="--set full --clock-control none --import-source on --profile-from-start off"
ncu $F -k regex:"fdm3_kernel<true, true>" -c 1 -o $O/fdm3_od python scripts/prof_solve.py c4 > $O/l1.log 2>&1
ncu $F -k regex:"fdm3_kernel<true, false>" -c 1 -o $O/fdm3 python scripts/prof_solve.py c4 > $O/l2.log 2>&1
ncu $F -k regex:k_offdiag -c 1 -o $O/offdiag python scripts/prof_solve.py c2 > $O/l3.log 2>&1
ncu $F -k regex:k_sweep_win -s 2 -c 1 -o $O/sweep_win python scripts/prof_solve.py c3 > $O/l4.log 2>&1
ncu $F -k regex:k_eblock2 -s 2 -c 1 -o $O/eblock2 python scripts/prof_solve.py c3 > $O/l5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slab3d_n4_persist -s 20 -c 1 \
    -o $O/slab3d python bench.py --steps 20 --warmup 5 --no-extra --no-cpu > $O/l6.log 2>&1
python scripts/ncu_summary.py $O/slab3d.ncu-rep $O/fdm3.ncu-rep $O/fdm3_od.ncu-rep \
    $O/offdiag.ncu-rep $O/sweep_win.ncu-rep $O/eblock2.ncu-rep > $O/ncu_summaries.md 2> $O/summary.err
echo done > $O/done
