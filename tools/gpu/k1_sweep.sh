#!/bin/bash
# K1 ring depth / chunk size sweep (64-layer batch, config-3 shape)
OUT=gpurun_out; mkdir -p $OUT
for nb in 1 2 3 4; do for ch in 8192 16384 32768; do
  echo "NBUF=$nb CHUNK=$ch: $(SCOUT_K1_NBUF=$nb SCOUT_K1_CHUNK=$ch timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done; done
