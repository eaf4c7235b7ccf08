#!/bin/bash
# Krylov combination variants under the power cap: 512 threads (default) vs 256, per-warp bulk copies
mkdir -p gpurun_out
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2ai_$TAG.json 2> gpurun_out/r2ai_$TAG.err; echo "$TAG rc=$?"; }
TAG=c512 run
RSV_LIB=$PWD/tools/_rsv_c256.so TAG=c256 run
RSV_LIB=$PWD/tools/_rsv_ctma.so TAG=ctma run
TAG=c512b run
RSV_LIB=$PWD/tools/_rsv_c256.so TAG=c256b run
