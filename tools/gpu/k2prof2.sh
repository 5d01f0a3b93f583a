for c in "--tier static" "--config qwen3-8b-16k --tier static" "--config qwen3-8b-16k"; do
  echo "== $c"
  SCOUT_K2_PROF=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $c 2>&1 >/dev/null | grep "k2 prof"
done
