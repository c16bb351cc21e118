#!/bin/bash
# usage: tools/build_full_variant.sh <name> [-DFOO=1 ...]
# Builds variants/<name>/libumcg.so from every source compiled with extra defines.
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
O=$R/variants/$name
mkdir -p $O
objs=""
for src in $(cd $R/paper_2501_06910_b200/csrc && ls *.cu | sed 's/\.cu$//'); do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Xcompiler -fopenmp --expt-relaxed-constexpr "$@" -c $R/paper_2501_06910_b200/csrc/$src.cu -o $O/$src.o &
  objs="$objs $O/$src.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $O/libumcg.so $objs -lcudart -lgomp
echo built variants/$name
