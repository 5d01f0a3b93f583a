#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02m}
timeout 600 python tools/debug/e2e_trace.py $OUT/e2e_trace_$TAG.json > $OUT/e2e_trace_$TAG.txt 2>&1
timeout 900 python tools/debug/layerwise_ctas.py 96 88 80 72 64 80 72 > $OUT/lw_ctas_$TAG.txt 2>&1
