#!/bin/bash
# One gpurun call: GPU parity suite, smoke, the bench (both arms), the config
# sweep, the ncu launch list and full captures of K2 / K1 / K6.
# Usage (repo root, on the GPU box): bash tools/gpu/round_check.sh <tag> [skip_tests]
set -x
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu_info_$TAG.txt
if [ "${2:-}" != "skip_tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
fi
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 2 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
# sweep (BASELINE configs; the f32 query / partial line; the stagger cadence; the kernel view)
timeout 600 python bench.py --recall-policy stagger --no-cpu-baseline > $OUT/sweep_stagger_$TAG.json 2> $OUT/sweep_stagger_$TAG.err
timeout 600 python bench.py --victim-cache off --no-extras --no-cpu-baseline > $OUT/sweep_novictim_$TAG.json 2> $OUT/sweep_novictim_$TAG.err
timeout 600 python bench.py --warm-seed off --no-extras --no-cpu-baseline > $OUT/sweep_noseed_$TAG.json 2> $OUT/sweep_noseed_$TAG.err
timeout 600 python bench.py --q-dtype f32 --cpu-dtype f32 --no-extras --no-cpu-baseline > $OUT/sweep_f32_$TAG.json 2> $OUT/sweep_f32_$TAG.err
timeout 600 python bench.py --config qwen3-8b-16k --no-cpu-baseline > $OUT/sweep_cfg2_$TAG.json 2> $OUT/sweep_cfg2_$TAG.err
timeout 600 python bench.py --config qwen3-32b-128k --no-cpu-baseline > $OUT/sweep_cfg5_$TAG.json 2> $OUT/sweep_cfg5_$TAG.err
timeout 600 python bench.py --config toy-4k-f32 --no-cpu-baseline --steps 256 > $OUT/sweep_cfg1_$TAG.json 2> $OUT/sweep_cfg1_$TAG.err
timeout 600 python bench.py --tier static --no-cpu-baseline > $OUT/sweep_static_$TAG.json 2> $OUT/sweep_static_$TAG.err
timeout 900 python bench.py --config qwen3-32b-32k-b128 --tier static --no-cpu-baseline > $OUT/sweep_cfg4_n1_$TAG.json 2> $OUT/sweep_cfg4_n1_$TAG.err
SCOUT_ENGINE_PHASES=1 timeout 300 python bench.py --steps 32 --warmup 3 --profile > /dev/null 2> $OUT/phases_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" -k "regex:score_topk|sparse_decode|decode_f32|combine|merge|recall|digest|kv_|tier|advance|writeback" -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --profile --steps 2 --warmup 1 > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:sparse_decode_tc -c 1 -f -o $OUT/prof_k2_$TAG \
  python bench.py --profile --steps 2 --warmup 1 > $OUT/ncu_k2_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:score_topk -c 1 -f -o $OUT/prof_k1_$TAG \
  python bench.py --profile --steps 2 --warmup 1 > $OUT/ncu_k1_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:qpred_gemm -s 2 -c 1 -f -o $OUT/prof_k6_$TAG \
  python tools/debug/qpred_once.py > $OUT/ncu_k6_$TAG.log 2>&1
timeout 300 python tools/debug/time_qpred.py > $OUT/time_qpred_$TAG.txt 2>&1
ls -la $OUT
