#!/bin/bash
export SCOUT_K1K2_OVERLAP=0  # the sanitizer serialises kernels: no K1 beside a K2 that waits for it
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-san3}
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_decode_scale.py tests/test_gpu_engine_tier.py tests/test_gpu_engine_worker.py tests/test_gpu_topk.py tests/test_gpu_tier.py"
timeout 3000 $CS --tool memcheck --print-limit 20 --error-exitcode 99 python -m pytest $T -q -x -p no:cacheprovider > $OUT/memcheck_$TAG.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck_$TAG.log
