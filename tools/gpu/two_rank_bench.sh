#!/bin/bash
# The N > 1 bench plumbing on one GPU: 2 ranks (gloo collectives, both on cuda:0), small shards.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02o}
export SCOUT_DIST_BACKEND=gloo SCOUT_BENCH_ONE_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --batch 2 --warm-slots 16 --steps 32 --warmup 3 --e2e-steps 16 --no-extras --no-cpu-baseline \
  > $OUT/bench_n2_$TAG.json 2> $OUT/bench_n2_$TAG.err; echo "rc=$?" >> $OUT/bench_n2_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --gpus 2 --global-batch 5 --warm-slots 16 --steps 32 --warmup 3 --e2e-steps 16 --no-extras --no-cpu-baseline \
  > $OUT/bench_n2s_$TAG.json 2> $OUT/bench_n2s_$TAG.err; echo "rc=$?" >> $OUT/bench_n2s_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $OUT/bench_n2ref_$TAG.json 2> $OUT/bench_n2ref_$TAG.err; echo "rc=$?" >> $OUT/bench_n2ref_$TAG.err
