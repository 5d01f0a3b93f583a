#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02j}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_topk -s 3 -c 1 -f -o $OUT/prof_k1one_$TAG python tools/debug/k1_one_layer.py > $OUT/ncu_k1one_$TAG.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score_topk --csv python tools/debug/k1_one_layer.py > $OUT/k1one_times_$TAG.csv 2>&1
timeout 600 python bench.py --tier static --no-cpu-baseline > $OUT/sweep_static_$TAG.json 2> $OUT/sweep_static_$TAG.err
