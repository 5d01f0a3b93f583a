#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02c2}
SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --config qwen3-8b-16k --steps 32 --warmup 3 --profile > /dev/null 2> $OUT/phases_cfg2_$TAG.err
SCOUT_K2_PROF=1 timeout 300 python bench.py --config qwen3-8b-16k --steps 32 --warmup 3 --profile > /dev/null 2> $OUT/k2prof_cfg2_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -c 200 --csv --log-file $OUT/launches_cfg2_$TAG.csv python bench.py --config qwen3-8b-16k --profile --steps 2 --warmup 1 > /dev/null 2>&1
