set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in "--config qwen3-8b-16k --tier static" "--tier static" "--config qwen3-32b-128k --tier static" ""; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'].get('workload'), d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved'], d['roofline'].get('k2_ms', ''))"
done
