#!/bin/bash
# K1 build-variant A/B (time_k1.py at the tier-mode stride), interleaved
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02p}
for r in 1 2 3; do for v in base dcb8minb4 minb5 minb7 dcb8; do
  echo "$v: $(SCOUT_B200_LIB=paper_2603_27138_b200/_ab/libscout_b200_$v.so NBS=520 NTOK=32801 timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done; done > $OUT/k1_variants_$TAG.txt 2>&1
