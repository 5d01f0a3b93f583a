#!/bin/bash
# Full GPU suite + smoke at HEAD.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02d}
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
SCOUT_LW_HOSTPROF=1 timeout 300 python tools/debug/time_layer_kernels.py > $OUT/lw_kernels_$TAG.txt 2>&1
