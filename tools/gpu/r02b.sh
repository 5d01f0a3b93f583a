#!/bin/bash
# Round-2 state check at HEAD: GPU suite, smoke, default bench (both cadences), phases.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02b}
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 40 --warmup 3 --profile > /dev/null 2> $OUT/phases_$TAG.err
