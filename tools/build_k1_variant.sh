#!/bin/bash
# Build a K1 variant library for an A/B run: k1_score_topk.cu recompiled with
# extra nvcc flags, linked with the other current objects.
#   tools/build_k1_variant.sh <name> <nvcc flags...>  -> paper_2603_27138_b200/_ab/libscout_b200_<name>.so
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
P=$R/paper_2603_27138_b200
name=$1; shift
mkdir -p $P/_ab /tmp/k1v
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC "$@" \
  -c $P/csrc/k1_score_topk.cu -o /tmp/k1v/k1_$name.o
objs=$(ls $P/_obj/*.o | grep -v k1_score_topk)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/_ab/libscout_b200_$name.so $objs /tmp/k1v/k1_$name.o -cudart static -Xcompiler -pthread
echo built $P/_ab/libscout_b200_$name.so
