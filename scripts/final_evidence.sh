#!/bin/bash
# Round-end evidence: default bench line, the bench's ncu launch list, one
# --set full capture of the headline kernel, and a c4 solve launch list.
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/ncu_bench_launches.csv \
    python bench.py --steps 50 --warmup 5 --no-extra --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu_bench.log
ncu -k regex:slab3d_n4_persist --set full --clock-control none --import-source on -s 20 -c 1 \
    -o gpurun_out/slab3d_full python bench.py --steps 50 --warmup 5 --no-extra --no-cpu \
    > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
ncu -i gpurun_out/slab3d_full.ncu-rep --page raw --csv > gpurun_out/slab3d_full_raw.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/ncu_c4_solve_launches.csv python scripts/prof_solve.py c4 \
    > gpurun_out/ncu_solve.log 2>&1
echo "ncu solve exit $?" >> gpurun_out/ncu_solve.log
ncu -k regex:fdm_kernel --set full --clock-control none --import-source on -c 1 \
    -o gpurun_out/fdm_full python scripts/prof_solve.py c4 > gpurun_out/ncu_fdm.log 2>&1
ncu -i gpurun_out/fdm_full.ncu-rep --page raw --csv > gpurun_out/fdm_full_raw.csv 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/ncu_c3_solve_launches.csv python scripts/prof_solve.py c3 \
    > gpurun_out/ncu_c3.log 2>&1
python bench.py --impl reference --steps 100 --warmup 2 > gpurun_out/ref.json 2>/dev/null
