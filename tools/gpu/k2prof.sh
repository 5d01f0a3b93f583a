# K2 cycle accounting (SCOUT_K2_PROF=1, printed at engine destroy) + a plain timing run
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "--tier static" "--config qwen3-8b-16k --tier static" "--config qwen3-32b-128k --tier static"; do
  echo "== $c"
  SCOUT_K2_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $c 2>&1 >/dev/null | grep "k2 prof"
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('step', round(d['ms_per_step'],3), 'k2', round(d['roofline']['avg_launch_us'],1), 'GB/s', round(d['roofline']['achieved']))"
done
