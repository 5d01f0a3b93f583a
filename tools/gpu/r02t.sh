#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02t}
timeout 1200 python tools/debug/layerwise_ctas.py -1 136 128 120 112 104 96 120 128 > $OUT/lw_ctas_$TAG.txt 2>&1
