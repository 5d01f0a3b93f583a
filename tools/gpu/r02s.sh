#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02s}
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_bench_scale.py -q -x > $OUT/pytest_k1_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_k1_$TAG.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score_topk --csv python tools/debug/k1_one_layer.py > $OUT/k1one_times_$TAG.csv 2>&1
for r in 1 2 3; do NBS=520 NTOK=32801 timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch; done > $OUT/k1_batch_$TAG.txt
timeout 900 python tools/debug/layerwise_ctas.py 80 96 80 > $OUT/lw_ctas_$TAG.txt 2>&1
