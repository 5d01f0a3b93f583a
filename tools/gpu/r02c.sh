#!/bin/bash
# Victim cache + SM-gather recalls: the tier / engine / bench-scale GPU tests, then the bench.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02c}
timeout 900 python -m pytest tests/test_gpu_tier.py tests/test_gpu_engine_tier.py tests/test_gpu_bench_scale.py -q -x > $OUT/pytest_tier_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_tier_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 40 --warmup 3 --profile > /dev/null 2> $OUT/phases_$TAG.err
