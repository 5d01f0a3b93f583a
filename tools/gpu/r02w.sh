#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02w}
timeout 900 python -m pytest tests/test_gpu_engine_tier.py tests/test_gpu_qpred.py -q -x > $OUT/pytest_lwq_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_lwq_$TAG.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
