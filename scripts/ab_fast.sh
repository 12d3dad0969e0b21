#!/bin/bash
# A/B of the fast-kernel variants + GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in 1 2; do
  STG_FAST_VARIANT=$v timeout 300 python bench.py --steps 8000 --no-cpu --no-extra > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err
done
