#!/bin/bash
# Round-2 (final session) evidence on the GPU box: the bench line and the
# reference arm, the ncu launch lists of the bench and of the c4 / c2 / c3
# solves, --set full captures of the headline R(U) and of the preconditioner
# kernels inside warm solves, and their markdown summary.
set -u
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/ev10; mkdir -p $O
T0=$SECONDS; python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench.py wall $((SECONDS - T0)) s" > $O/bench_time.txt
python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err
python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/ncu_bench_launches.csv python bench.py --steps 20 --warmup 5 --no-extra --no-cpu \
    > $O/ncu_bench.log 2>&1
for c in c4 c2 c3 c5; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $O/ncu_${c}_solve_launches.csv python scripts/prof_solve.py $c \
      > $O/ncu_${c}_solve.log 2>&1
done
F="--set full --clock-control none --import-source on --profile-from-start off"
ncu $F -k regex:fdm3_kernel -c 1 -o $O/fdm3 python scripts/prof_solve.py c4 > $O/l1.log 2>&1
ncu $F -k regex:fdm3_kernel -s 1 -c 1 -o $O/fdm3_coupled python scripts/prof_solve.py c4 > $O/l2.log 2>&1
ncu $F -k regex:fdm2i_kernel -s 1 -c 1 -o $O/fdm2i_coupled python scripts/prof_solve.py c2 > $O/l3.log 2>&1
ncu $F -k regex:k_sweep_win -s 2 -c 1 -o $O/sweep_win python scripts/prof_solve.py c3 > $O/l4.log 2>&1
STG_PRECOND_LAG_STEPS=1 ncu $F -k regex:k_build_burgers -c 1 -o $O/build_blocks python scripts/prof_solve.py c3 > $O/l5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:slab3d_n4_persist -s 20 -c 1 \
    -o $O/slab3d python bench.py --steps 20 --warmup 5 --no-extra --no-cpu > $O/l6.log 2>&1
echo done > $O/done
