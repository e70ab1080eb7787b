#!/bin/bash
# Build librsim variants with different compile-time tuning macros for one
# source (SRC, default krylov.cu) into paper_2008_01539_b200/lib/ab/librsim_<name>.so
# (A/B experiments; load with RSIM_LIB=...).
# Usage: [SRC=krylov_dsm.cu] scripts/ab_krylov_build.sh name "-DMACRO=v ..." ...
set -e
cd "$(dirname "$0")/.."
OBJ=paper_2008_01539_b200/lib/obj
OUT=paper_2008_01539_b200/lib/ab
mkdir -p $OUT
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -ccbin /usr/bin/g++ -Xcompiler -fPIC,-ffp-contract=off,-fopenmp,-O3 -Xptxas -O3 -I include -I paper_2008_01539_b200/csrc"
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  src=${SRC:-krylov.cu}
  $NV $flags -c paper_2008_01539_b200/csrc/$src -o $OUT/v_$name.o
  objs=$(ls $OBJ/*.o | grep -v "/$src.o")
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ $objs $OUT/v_$name.o -o $OUT/librsim_$name.so -lgomp
  rm -f $OUT/v_$name.o
  echo built $OUT/librsim_$name.so
done
