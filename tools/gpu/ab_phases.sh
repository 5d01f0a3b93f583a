# A/B of tier-mode phase times: built library ("new") vs libscout_b200_old.so ("alt")
L=paper_2603_27138_b200
cp $L/libscout_b200.so /tmp/new.so
for v in new alt new alt; do
  if [ $v = new ]; then cp /tmp/new.so $L/libscout_b200.so; else cp $L/libscout_b200_old.so $L/libscout_b200.so; fi
  echo "== $v"; SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 14 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "^step" | tail -4
done
cp /tmp/new.so $L/libscout_b200.so
