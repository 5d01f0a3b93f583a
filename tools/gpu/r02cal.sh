#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02cal}
timeout 600 python -m pytest tests/test_gpu_engine_tier.py -q -x -k "cpu_tokens" > $OUT/pytest_cal_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_cal_$TAG.log
timeout 900 python bench.py --recall-calibrate 24 --no-extras --no-cpu-baseline > $OUT/bench_cal_$TAG.json 2> $OUT/bench_cal_$TAG.err
