#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
SCOUT_K2_PROF=1 timeout 300 python tools/debug/layerwise_dev.py > $OUT/g15_prof.txt 2>&1
SCOUT_K1_DIRECT=0 SCOUT_K1_NBUF=3 SCOUT_K1_CHUNK=32768 timeout 300 python tools/debug/layerwise_dev.py > $OUT/g15_ring3.txt 2>&1
SCOUT_K1_DIRECT=0 SCOUT_K1_NBUF=4 SCOUT_K1_CHUNK=65536 timeout 300 python tools/debug/layerwise_dev.py > $OUT/g15_ring4.txt 2>&1
