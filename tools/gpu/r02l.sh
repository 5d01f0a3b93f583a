#!/bin/bash
# K1 L2-prefetch A/B (env knobs on one library): fused batch at the tier stride, single layer, in-step phases
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02l}
for r in 1 2; do
for pf in 0 8 16 32 64; do for pft in 0 1; do
  echo "PF=$pf PFT=$pft: $(SCOUT_K1_PF=$pf SCOUT_K1_PFT=$pft NBS=520 NTOK=32801 timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done; done
done > $OUT/k1_pf_$TAG.txt 2>&1
for pf in 0 16; do for pft in 0 1; do
  echo "PF=$pf PFT=$pft: $(SCOUT_K1_PF=$pf SCOUT_K1_PFT=$pft timeout 120 python tools/debug/time_layer_kernels.py 2>&1 | grep K1)"
done; done >> $OUT/k1_pf_$TAG.txt 2>&1
for pf in 0 16; do
  SCOUT_K1_PF=$pf SCOUT_K1_PFT=$pf SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 32 --warmup 3 --profile > /dev/null 2> $OUT/phases_pf${pf}_$TAG.err
done
