# A/B in tier mode (K1 phase + step): built library ("new") vs libscout_b200_old.so ("old")
L=paper_2603_27138_b200
cp $L/libscout_b200.so /tmp/new.so
for v in new old new old new old; do
  if [ $v = new ]; then cp /tmp/new.so $L/libscout_b200.so; else cp $L/libscout_b200_old.so $L/libscout_b200.so; fi
  k1=$(SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 12 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep '^step' | grep plan | awk '{print $6}' | sort -n | head -4 | tr '\n' ' ')
  st=$(timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3))")
  echo "$v K1: $k1 step: $st"
done
cp /tmp/new.so $L/libscout_b200.so
