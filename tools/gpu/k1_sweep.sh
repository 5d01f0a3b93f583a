#!/bin/bash
# K1 ring depth / chunk size sweep (64-layer batch, config-3 shape)
OUT=gpurun_out; mkdir -p $OUT
for cfg in "2 8192" "2 4096" "3 4096" "3 8192" "4 4096" "4 8192" "3 16384" "2 16384"; do
  set -- $cfg
  echo "NBUF=$1 CHUNK=$2: $(SCOUT_K1_NBUF=$1 SCOUT_K1_CHUNK=$2 timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done
