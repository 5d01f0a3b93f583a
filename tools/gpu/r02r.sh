#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02r}
SCOUT_B200_LIB=paper_2603_27138_b200/_ab/libscout_b200_trace.so timeout 120 python tools/debug/k1_one_layer.py > $OUT/k1_trace_one_$TAG.txt 2>&1
