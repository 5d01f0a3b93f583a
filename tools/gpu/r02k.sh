#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02k}
timeout 900 python -m pytest tests/test_gpu_cpp_tier.py tests/test_gpu_tier.py tests/test_gpu_cpp_wrapper.py tests/test_gpu_dropin_engine.py -q -x -s > $OUT/pytest_cpptier_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_cpptier_$TAG.log
