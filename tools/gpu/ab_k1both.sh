# A/B of K1 (built library "new" vs libscout_b200_old.so "old"): parity, K1 alone (static shape), tier K1 phase + step
L=paper_2603_27138_b200
timeout 600 python -m pytest tests/test_gpu_topk.py tests/test_gpu_engine_tier.py -x -q 2>&1 | tail -1
cp $L/libscout_b200.so /tmp/new.so
for v in new old new old; do
  if [ $v = new ]; then cp /tmp/new.so $L/libscout_b200.so; else cp $L/libscout_b200_old.so $L/libscout_b200.so; fi
  k1s=$(timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch | awk '{print $3}')
  k1=$(SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 12 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep '^step' | grep plan | awk '{print $6}' | sort -n | head -4 | tr '\n' ' ')
  st=$(timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))")
  echo "$v K1 static: $k1s  tier K1: $k1 tier step: $st"
done
cp /tmp/new.so $L/libscout_b200.so
