#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02g}
timeout 300 python tools/debug/cpu_unit_cost.py > $OUT/cpu_unit_cost_$TAG.txt 2>&1
SCOUT_CW_PROF=1 timeout 900 python tools/debug/e2e_worker_dtypes.py > $OUT/e2e_worker_dtypes_$TAG.txt 2> $OUT/cw_prof_$TAG.txt
