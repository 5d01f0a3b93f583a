#!/bin/bash
# PCIe recall microbench + the recall burst at the reference cadence (ce / sm)
OUT=gpurun_out; mkdir -p $OUT
timeout 300 ./tools/microbench/pcie_recall 48000 > $OUT/pcie_recall.txt 2>&1
timeout 300 ./tools/microbench/pcie_recall 6000 >> $OUT/pcie_recall.txt 2>&1
for m in ce sm; do
SCOUT_RECALL_PROF=1 SCOUT_ENGINE_PHASES=1 timeout 600 python bench.py --no-extras --no-cpu-baseline --recall-mode $m --steps 32 > $OUT/g11_$m.json 2> $OUT/g11_$m.err
done
