#!/bin/bash
export SCOUT_K1K2_OVERLAP=0  # the sanitizer serialises kernels: no K1 beside a K2 that waits for it
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-san2}
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_engine.py tests/test_gpu_kv_merge_recall.py tests/test_gpu_engine_tier.py::test_engine_layerwise_with_query_prediction tests/test_gpu_qpred.py::test_predict_query_vs_reference"
timeout 3000 $CS --tool memcheck --print-limit 20 --error-exitcode 99 python -m pytest $T -q -x -p no:cacheprovider -k "not 40" > $OUT/memcheck_$TAG.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck_$TAG.log
