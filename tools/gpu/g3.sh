timeout 1200 python -m pytest tests/test_gpu_engine_worker.py tests/test_gpu_engine_tier.py tests/test_gpu_engine.py -x -q -m gpu 2>&1 | tail -30
