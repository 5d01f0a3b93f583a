#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
for c in 0 136 128 116; do
SCOUT_LW_K2_CTAS=$c timeout 300 python tools/debug/layerwise_dev.py > $OUT/g16_c$c.txt 2>&1
done
SCOUT_LW_K2_CTAS=128 SCOUT_K1_DIRECT=0 SCOUT_K1_NBUF=3 SCOUT_K1_CHUNK=32768 timeout 300 python tools/debug/layerwise_dev.py > $OUT/g16_c128_ring3.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_engine_tier.py tests/test_gpu_decode_scale.py tests/test_gpu_decode.py -q -m gpu -x > $OUT/g16_pytest.txt 2>&1
