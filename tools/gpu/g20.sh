#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_topk.py tests/test_gpu_engine_tier.py tests/test_gpu_bench_scale.py -q -m gpu -x > $OUT/g20_pytest.txt 2>&1
timeout 300 python tools/debug/time_layer_kernels.py > $OUT/g20_iso.txt 2>&1
for c in 0 128 120 112; do
SCOUT_LW_K2_CTAS=$c timeout 300 python tools/debug/layerwise_dev.py > $OUT/g20_c$c.txt 2>&1
done
