#!/bin/bash
# K2 plan-buffer variants: config 2 / config 3 steps (interleaved) + K2 tests on the 3-plan variant
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02k2}
SCOUT_B200_LIB=paper_2603_27138_b200/_ab/libscout_b200_p3s32b256.so timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_decode_scale.py tests/test_gpu_engine.py tests/test_gpu_engine_tier.py -q -x > $OUT/pytest_k2v_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_k2v_$TAG.log
for r in 1 2; do for v in base p3s32b256 p2s32b256; do
  for cfg in qwen3-8b-16k qwen3-32b-32k; do
    echo "$v $cfg: $(SCOUT_B200_LIB=paper_2603_27138_b200/_ab/libscout_b200_$v.so timeout 300 python bench.py --config $cfg --steps 32 --warmup 3 --profile 2>&1 | grep '^step ' | tail -1)"
  done
done; done > $OUT/k2_variants_$TAG.txt 2>&1
