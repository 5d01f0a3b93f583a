set -x
timeout 900 python -m pytest tests/test_gpu_engine_tier.py tests/test_gpu_engine.py -x -q -m gpu 2>&1 | tail -30
for pol in reference stagger; do
timeout 600 python bench.py --steps 64 --warmup 5 --no-cpu-baseline --recall-policy $pol > gpurun_out/g2_bench_$pol.json 2> gpurun_out/g2_bench_$pol.err; tail -2 gpurun_out/g2_bench_$pol.err
done
