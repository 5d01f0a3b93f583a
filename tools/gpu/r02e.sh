#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02e}
nproc > $OUT/cpuw_$TAG.txt; lscpu | grep -E "Model name|Thread|Core|Socket|L3|NUMA" >> $OUT/cpuw_$TAG.txt
timeout 600 python tools/debug/cpu_worker_probe.py >> $OUT/cpuw_$TAG.txt 2>&1
timeout 300 python tools/debug/layerwise_trace.py $OUT/lw_trace_$TAG.json > $OUT/lw_trace_$TAG.txt 2>&1
