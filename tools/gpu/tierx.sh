# tier-mode change check: tier parity tests, phases, bench (tier and static)
timeout 900 python -m pytest tests/test_gpu_engine_tier.py tests/test_gpu_tier.py tests/test_gpu_engine.py -x -q 2>&1 | tail -2
SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 14 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "^step" | tail -6
for r in 1 2; do for c in "" "--tier static"; do
  timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tier' if d.get('tier') else 'static', 'step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), 'k2', round(d['roofline']['avg_launch_us'],1), 'launches', d['gpu_launches'])"
done; done
