#!/bin/bash
# GPU tests, then per-config warm solve times and kernel timelines for c4 c2 c5 c3.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in c4 c2 c5 c3; do
  echo "== $c"; timeout 120 python scripts/prof_solve.py $c 2>&1 | grep -v Warn
  timeout 120 python scripts/solve_timeline.py $c 2>&1 | grep config
done > gpurun_out/solve.log 2>&1
