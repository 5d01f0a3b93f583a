timeout 900 python -m pytest tests/test_gpu_bench_scale.py -x -q -m gpu 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err; echo rc=$?; tail -8 gpurun_out/g7_bench.err
