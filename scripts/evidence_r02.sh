#!/bin/bash
# Round-2 evidence (run on the GPU box): bench line, its ncu launch list, one
# --set full capture each of the headline kernel and the FDM kernels, the
# c4 / c2 / c3 solve launch lists, the reference arm.
set -u
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/ev
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/ref.json 2> $O/ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/ncu_bench_launches.csv \
    python bench.py --steps 20 --warmup 5 --no-extra --no-cpu > $O/ncu_bench.log 2>&1
ncu -k regex:slab3d_n4_persist --set full --clock-control none --import-source on -s 20 -c 1 \
    -o $O/slab3d_full python bench.py --steps 20 --warmup 5 --no-extra --no-cpu \
    > $O/ncu_full.log 2>&1
for c in c4 c2 c3; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file $O/ncu_${c}_solve_launches.csv python scripts/prof_solve.py $c \
      > $O/ncu_${c}_solve.log 2>&1
done
ncu -k regex:fdm3_kernel --set full --clock-control none --import-source on -s 3 -c 1 \
    -o $O/fdm3_full python scripts/fdm_graph_bench.py c4 > $O/ncu_fdm3.log 2>&1
ncu -k regex:fdm2_kernel --set full --clock-control none --import-source on -s 3 -c 1 \
    -o $O/fdm2_full python scripts/fdm_graph_bench.py c2 > $O/ncu_fdm2.log 2>&1
for f in slab3d_full fdm3_full fdm2_full; do
  ncu -i $O/$f.ncu-rep --page raw --csv > $O/${f}_raw.csv 2>&1
done
echo done > $O/done
