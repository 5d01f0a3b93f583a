#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python tools/debug/time_layer_kernels.py > $OUT/g17_direct.txt 2>&1
SCOUT_K1_DIRECT=0 SCOUT_K1_NBUF=3 SCOUT_K1_CHUNK=32768 timeout 300 python tools/debug/time_layer_kernels.py > $OUT/g17_ring3.txt 2>&1
SCOUT_K1_DIRECT=0 SCOUT_K1_NBUF=4 SCOUT_K1_CHUNK=49152 timeout 300 python tools/debug/time_layer_kernels.py > $OUT/g17_ring4.txt 2>&1
SCOUT_K2_PROF=1 SCOUT_LW_K2_CTAS=128 timeout 300 python tools/debug/layerwise_dev.py > $OUT/g17_prof.txt 2>&1
