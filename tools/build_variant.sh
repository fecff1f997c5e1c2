#!/bin/bash
# Build a variant of libpaco_b200.so with tc_gemm.cu recompiled under extra -D
# flags (kernel-configuration experiments; load it with PACO_LIB=<path>).
#   tools/build_variant.sh <name> -DPACO_EPI_RING=1 -DPACO_RES_AST=4 ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
OBJ=$ROOT/paper_2011_01441_b200/build_obj
OUT=$ROOT/variants
mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include "$@" \
     -c $ROOT/paper_2011_01441_b200/csrc/tc_gemm.cu -o $OUT/tc_gemm_$name.o
objs=$(ls $OBJ/*.o | grep -v '/tc_gemm.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libpaco_$name.so $objs $OUT/tc_gemm_$name.o
echo $OUT/libpaco_$name.so
