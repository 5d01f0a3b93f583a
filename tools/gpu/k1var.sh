# K1 direct-load variants (libscout_b200_v{A,B,C}.so): K1 alone (static shape) and tier-mode K1 phase
L=paper_2603_27138_b200
cp $L/libscout_b200.so /tmp/cur.so
for r in 1 2; do for v in B D; do
  cp $L/libscout_b200_v$v.so $L/libscout_b200.so
  echo "$v: $(timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch) | tier K1: $(SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 12 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep '^step' | tail -6 | awk '{print $6}' | sort -n | head -3 | tr '\n' ' ')"
done; done
cp /tmp/cur.so $L/libscout_b200.so
