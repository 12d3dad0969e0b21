#!/bin/bash
# A/B of the fdm3 segment size (STG_FDM3_E / STG_FDM3_MINB variants built by
# scripts/build_variant.sh): the plain apply in a CUDA graph and warm solves
# (c4 / c5 / c2 / c3), interleaved over two rounds.
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/fdm3e; mkdir -p $O
for r in 1 2; do
  for v in base "$@"; do
    lib=""; [ "$v" != base ] && lib=scripts/variants/$v/libstg_cuda.so
    STG_CUDA_LIB=$lib python scripts/fdm_graph_bench.py c4 > $O/fdm_${v}_$r.json 2>&1
    STG_CUDA_LIB=$lib python scripts/warm_solves.py > $O/warm_${v}_$r.json 2>&1
  done
done
