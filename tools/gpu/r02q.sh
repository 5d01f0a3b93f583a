#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02q}
for r in 1 2 3 4; do for v in base minb7 minb8; do
  echo "$v: $(SCOUT_B200_LIB=paper_2603_27138_b200/_ab/libscout_b200_$v.so NBS=520 NTOK=32801 timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done; done > $OUT/k1_variants_$TAG.txt 2>&1
for v in base minb7 minb8; do
  SCOUT_B200_LIB=paper_2603_27138_b200/_ab/libscout_b200_$v.so SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 32 --warmup 3 --profile > /dev/null 2> $OUT/phases_${v}_$TAG.err
done
