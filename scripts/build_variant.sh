#!/bin/bash
# Build an A/B variant of libstg_cuda.so with extra nvcc defines into
# scripts/variants/<name>/ (load it with STG_CUDA_LIB=<path>).
#   scripts/build_variant.sh <name> -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=scripts/variants/$name
mkdir -p $out
objs=""
for f in kernels_slab kernels_vec kernels_precond kernels_fdm kernels_general kernels_small; do
  nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude "$@" \
    -c paper_2201_05800_b200/csrc/$f.cu -o $out/$f.o &
  objs="$objs $out/$f.o"
done
nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude "$@" -c paper_2201_05800_b200/csrc/stg.cpp -o $out/stg.o &
wait
nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -shared -o $out/libstg_cuda.so $objs $out/stg.o
rm -f $out/*.o
echo $out/libstg_cuda.so
