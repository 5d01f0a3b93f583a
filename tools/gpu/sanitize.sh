#!/bin/bash
export SCOUT_K1K2_OVERLAP=0  # the sanitizer serialises kernels: no K1 beside a K2 that waits for it
# compute-sanitizer over small GPU tests: memcheck (out-of-bounds / misaligned
# accesses) and racecheck (shared-memory hazards) of the K1 / K2 / K5 kernels
# and the engine's device tier mode. Small shapes: the tools slow kernels ~100x.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-san}
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_tier.py tests/test_gpu_topk.py::test_topk_bit_exact_vs_reference_golden tests/test_gpu_topk.py::test_topk_band_edges_vs_oracle tests/test_gpu_decode.py tests/test_gpu_engine_tier.py::test_engine_victim_cache_matches_copies"
timeout 2400 $CS --tool memcheck --print-limit 20 --error-exitcode 99 python -m pytest $T -q -x -p no:cacheprovider > $OUT/memcheck_$TAG.log 2>&1; echo "memcheck rc=$?" >> $OUT/memcheck_$TAG.log
timeout 2400 $CS --tool racecheck --print-limit 20 --error-exitcode 99 python -m pytest tests/test_gpu_tier.py tests/test_gpu_topk.py::test_topk_bit_exact_vs_reference_golden tests/test_gpu_topk.py::test_topk_band_edges_vs_oracle -q -x -p no:cacheprovider > $OUT/racecheck_$TAG.log 2>&1; echo "racecheck rc=$?" >> $OUT/racecheck_$TAG.log
