#!/bin/bash
# Build a variant library for an A/B run: one csrc source recompiled with extra
# nvcc flags, linked with the other current objects.
#   tools/build_variant.sh <name> <source.cu> <nvcc flags...>  -> paper_2603_27138_b200/_ab/libscout_b200_<name>.so
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2603_27138_b200
name=$1; src=$2; shift 2
base=$(basename $src .cu)
mkdir -p $P/_ab /tmp/variants
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC "$@" \
  -c $P/csrc/$src -o /tmp/variants/${base}_$name.o
objs=$(ls $P/_obj/*.o | grep -v "/$base.cu.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/_ab/libscout_b200_$name.so $objs /tmp/variants/${base}_$name.o -cudart static -Xcompiler -pthread
echo built $P/_ab/libscout_b200_$name.so
