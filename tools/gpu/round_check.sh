#!/bin/bash
# One gpurun call: GPU parity suite, smoke, bench (both arms), ncu launch list + full captures.
# Usage (from the repo root, on the GPU box): bash tools/gpu/round_check.sh <tag> [skip_tests]
set -x
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu_info_$TAG.txt
if [ "${2:-}" != "skip_tests" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
fi
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 400 python bench.py --tier static > $OUT/bench_static_$TAG.json 2> $OUT/bench_static_$TAG.err
SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 30 --warmup 3 --profile > /dev/null 2> $OUT/phases_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k "regex:score_topk|sparse_decode|decode_f32|combine|merge|recall|digest|kv_|tier|advance|writeback" -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --profile --steps 2 --warmup 1 > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:sparse_decode_tc -c 1 -f -o $OUT/prof_k2_$TAG \
  python bench.py --profile --steps 2 --warmup 1 > $OUT/ncu_k2_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:score_topk -c 1 -f -o $OUT/prof_k1_$TAG \
  python bench.py --profile --steps 2 --warmup 1 > $OUT/ncu_k1_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qpred_gemm -s 2 -c 1 -f -o $OUT/prof_k6_$TAG \
  python tools/debug/qpred_once.py > $OUT/ncu_k6_$TAG.log 2>&1
timeout 300 python tools/debug/time_qpred.py > $OUT/time_qpred_$TAG.txt 2>&1
timeout 300 python tools/debug/e2e_probe.py > $OUT/e2e_probe_$TAG.txt 2>&1
ls -la $OUT
