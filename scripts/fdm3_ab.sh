#!/bin/bash
# A/B of fdm3_kernel: the in-tree build against scripts/variants/fdm_old
# (device time in a CUDA graph, c4), then the FDM exactness and c4 solve tests.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/fdm3ab; mkdir -p $O
for k in 1 2; do
  python scripts/fdm_graph_bench.py c4 > $O/new_$k.json 2>&1
  STG_CUDA_LIB=scripts/variants/fdm_old/libstg_cuda.so python scripts/fdm_graph_bench.py c4 > $O/old_$k.json 2>&1
done
python -m pytest tests -m gpu -x -q -k "fdm or element_block or solve or c5 or c4" > $O/pytest.log 2>&1
python scripts/solve_bench.py c4 c5 > $O/solve_new.json 2>&1
STG_CUDA_LIB=scripts/variants/fdm_old/libstg_cuda.so python scripts/solve_bench.py c4 c5 > $O/solve_old.json 2>&1
