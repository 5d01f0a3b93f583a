#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02v}
timeout 900 python bench.py --warm-seed off --warmup 40 --no-extras --no-cpu-baseline > $OUT/sweep_noseed_w40_$TAG.json 2> $OUT/sweep_noseed_w40_$TAG.err
timeout 900 python bench.py --steps 128 --no-extras --no-cpu-baseline > $OUT/sweep_s128_$TAG.json 2> $OUT/sweep_s128_$TAG.err
