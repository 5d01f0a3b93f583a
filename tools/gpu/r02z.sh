#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02z}
timeout 1200 python -m pytest tests/test_gpu_engine_tier.py -q -x > $OUT/pytest_f32eng_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_f32eng_$TAG.log
