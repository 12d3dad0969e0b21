#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload c2 --steps 2000 --no-cpu --no-extra > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
STG_2D_NONPERSIST=1 timeout 300 python bench.py --workload c2 --steps 1000 --no-cpu --no-extra > gpurun_out/bench_c2_np.json 2>/dev/null
python scripts/solve_bench.py c2 > gpurun_out/solve_c2.json 2>&1
