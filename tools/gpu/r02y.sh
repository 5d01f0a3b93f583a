#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02y}
timeout 300 python tools/debug/cpu_unit_cost.py > $OUT/cpu_unit_cost_$TAG.txt 2>&1
