#!/bin/bash
# usage: tools/build_variant.sh <name> <file.cu> [-DFOO=1 ...]
# Builds variants/<name>/libumcg.so from the current objects with <file.cu>
# recompiled under extra defines (for A/B timing with UMCG_LIB_PATH).
set -e
name=$1; src=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2501_06910_b200/_build
mkdir -p $R/variants/$name
obj=$R/variants/$name/$(basename $src .cu).o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Xcompiler -fopenmp --expt-relaxed-constexpr "$@" -c $R/paper_2501_06910_b200/csrc/$src -o $obj
objs=""
for o in $B/*.o; do
  if [ "$(basename $o)" == "$(basename $obj)" ]; then objs="$objs $obj"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/variants/$name/libumcg.so $objs -lcudart -lgomp
echo built variants/$name
