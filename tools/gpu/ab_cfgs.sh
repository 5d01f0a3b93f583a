# A/B over configs (static): built library ("new") vs libscout_b200_old.so ("old"), plus parity tests and K2 accounting
L=paper_2603_27138_b200
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_engine_tier.py -x -q 2>&1 | tail -1
cp $L/libscout_b200.so /tmp/new.so
for c in "--config qwen3-8b-16k --tier static" "--config qwen3-32b-128k --tier static" "--tier static" ""; do
  for v in new old new old; do
    if [ $v = new ]; then cp /tmp/new.so $L/libscout_b200.so; else cp $L/libscout_b200_old.so $L/libscout_b200.so; fi
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], 'tier' if d.get('tier') else 'static', 'step', round(d['ms_per_step'],3), 'k2', round(d['roofline']['avg_launch_us'],1))"
  done
done
cp /tmp/new.so $L/libscout_b200.so
for c in "--config qwen3-8b-16k --tier static" "--tier static"; do
  SCOUT_K2_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $c 2>&1 >/dev/null | grep "k2 prof"
done
