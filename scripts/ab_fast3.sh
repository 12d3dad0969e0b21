#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
for m in 2 3; do
  STG_FAST_CTAS_PER_SM=$m timeout 300 python bench.py --steps 8000 --no-cpu --no-extra > gpurun_out/bench_m$m.json 2>gpurun_out/bench_m$m.err
done
