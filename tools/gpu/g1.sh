set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_decode_scale.py tests/test_gpu_decode.py tests/test_gpu_engine.py tests/test_gpu_engine_tier.py -x -q -m gpu 2>&1 | tail -30
timeout 600 python bench.py --steps 32 --warmup 5 --no-cpu-baseline > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; tail -3 gpurun_out/g1_bench.err
