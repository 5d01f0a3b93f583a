# A/B: the built library vs libscout_b200_old.so, alternating, same box
L=paper_2603_27138_b200
cp $L/libscout_b200.so /tmp/new.so
for r in 1 2; do
for v in new old; do
  cp /tmp/$v.so $L/libscout_b200.so 2>/dev/null || cp $L/libscout_b200_old.so $L/libscout_b200.so
  [ $v = old ] && cp $L/libscout_b200_old.so $L/libscout_b200.so
  for c in "--tier static" ""; do
    timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'tier' if d.get('tier') else 'static', 'step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'k2', round(d['roofline']['avg_launch_us'],1))"
  done
done
done
cp /tmp/new.so $L/libscout_b200.so
