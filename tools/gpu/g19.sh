#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/g19_pytest.txt 2>&1
SCOUT_LW_HOSTPROF=1 SCOUT_LW_K2_CTAS=128 timeout 300 python tools/debug/layerwise_host.py > $OUT/g19_host.txt 2>&1
for c in 0 136 128 120; do
SCOUT_LW_K2_CTAS=$c timeout 300 python tools/debug/layerwise_dev.py > $OUT/g19_c$c.txt 2>&1
done
