#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02i}
timeout 600 python bench.py --tier static --no-cpu-baseline > $OUT/sweep_static_$TAG.json 2> $OUT/sweep_static_$TAG.err
timeout 900 python bench.py --config qwen3-32b-32k-b128 --tier static --no-cpu-baseline > $OUT/sweep_cfg4_n1_$TAG.json 2> $OUT/sweep_cfg4_n1_$TAG.err
timeout 900 python tools/debug/layerwise_ctas.py > $OUT/lw_ctas_$TAG.txt 2>&1
