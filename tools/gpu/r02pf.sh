#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02pf}
timeout 900 python -m pytest tests/test_gpu_tier.py -q -x > $OUT/pytest_prefill_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_prefill_$TAG.log
