#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02f}
g++ -O3 -march=native -fopenmp -o /tmp/host_bw tools/microbench/host_bw.cpp && /tmp/host_bw > $OUT/host_bw_$TAG.txt 2>&1
timeout 900 python tools/debug/e2e_worker_threads.py > $OUT/e2e_worker_threads_$TAG.txt 2>&1
