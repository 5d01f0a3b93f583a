#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02x}
for nst in 5 2; do
  echo "NST=$nst: $(SCOUT_QP_NST=$nst timeout 300 python tools/debug/time_qpred.py 2>&1 | tail -2 | tr '\n' ' ')"
  SCOUT_QP_NST=$nst timeout 900 python tools/debug/layerwise_qpred.py 2>&1 | grep layerwise | sed "s/^/NST=$nst /"
done > $OUT/lwq_nst_$TAG.txt 2>&1
