#!/bin/bash
# how many of the lowest bits the lo pass delegates to the mid pass (3 = default)
mkdir -p gpurun_out
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2ah_$TAG.json 2> gpurun_out/r2ah_$TAG.err; echo "$TAG rc=$?"; }
TAG=d3 run
RSV_LIB=$PWD/tools/_rsv_d2.so TAG=d2 run
RSV_LIB=$PWD/tools/_rsv_d1.so TAG=d1 run
TAG=d3b run
RSV_LIB=$PWD/tools/_rsv_d2.so TAG=d2b run
