timeout 900 python -m pytest tests/test_gpu_engine_tier.py -x -q -m gpu -k "layerwise" 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo rc=$?; tail -9 gpurun_out/g10_bench.err
