#!/bin/bash
# Device time of one bench script across A/B builds (scripts/variants/<name>):
#   scripts/variant_ab.sh <out-dir> "<script and args>" name1 name2 ...
# (the in-tree build runs as "tree"); two passes, interleaved.
cd "$(dirname "$0")/.." || exit 1
O=$1; shift; CMD=$1; shift
mkdir -p $O
for pass in 1 2; do
  python $CMD > $O/tree_$pass.json 2>&1
  for v in "$@"; do
    STG_CUDA_LIB=scripts/variants/$v/libstg_cuda.so python $CMD > $O/${v}_$pass.json 2>&1
  done
done
for f in $O/*.json; do echo "$f $(tail -1 $f)"; done
