#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02lw}
timeout 1500 python tools/debug/layerwise_ctas.py 80 96 112 128 -1 80 96 112 128 -1 80 96 112 128 -1 > $OUT/lw_ctas_$TAG.txt 2>&1
