#!/bin/bash
mkdir -p gpurun_out
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2ac_$TAG.json 2> gpurun_out/r2ac_$TAG.err; echo "$TAG rc=$?"; }
TAG=last run
RSV_LIB=$PWD/tools/_rsv_noshfl.so TAG=lds run
RSV_LIB=$PWD/tools/_rsv_tma8.so TAG=tma8 run
TAG=last2 run
RSV_LIB=$PWD/tools/_rsv_noshfl.so TAG=lds2 run
RSV_LIB=$PWD/tools/_rsv_tma8.so TAG=tma82 run
