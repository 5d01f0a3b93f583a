# K1 direct-load variant (SCOUT_K1_DIRECT=1) vs the bulk-copy ring: parity + timing
SCOUT_K1_DIRECT=1 timeout 600 python -m pytest tests/test_gpu_topk.py tests/test_gpu_engine.py tests/test_gpu_engine_tier.py -x -q 2>&1 | tail -2
for r in 1 2; do for d in 0 1; do
  echo "direct=$d: $(SCOUT_K1_DIRECT=$d timeout 120 python tools/debug/time_k1.py 2>&1 | grep batch)"
done; done
for d in 0 1 0 1; do
  echo "== tier phases direct=$d"; SCOUT_K1_DIRECT=$d SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 14 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "^step" | tail -3
done
for d in 0 1; do
  SCOUT_K1_DIRECT=$d timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct=$d tier step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
  SCOUT_K1_DIRECT=$d timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --tier static 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('direct=$d static step', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3))"
done
