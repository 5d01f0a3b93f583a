# K2 L2-prefetch distance sweep (SCOUT_K2_L2PF), static config 3 / 5 / 2
for c in "--tier static" "--config qwen3-32b-128k --tier static" "--config qwen3-8b-16k --tier static"; do
  for pf in 0 2 4 8 12; do
    SCOUT_K2_L2PF=$pf timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c pf=$pf', 'step', round(d['ms_per_step'],3), 'k2', round(d['roofline']['avg_launch_us'],1), 'GB/s', round(d['roofline']['achieved']))"
  done
done
SCOUT_K2_L2PF=4 SCOUT_K2_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --tier static 2>&1 >/dev/null | grep "k2 prof"
