#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r02n}
timeout 600 python tools/debug/e2e_vs_device.py > $OUT/e2e_vs_device_$TAG.txt 2>&1
