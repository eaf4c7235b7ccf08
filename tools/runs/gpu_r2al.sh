#!/bin/bash
# with the 256-thread lo pass: lowest bits delegated to the mid pass, 3 (default) vs 2
mkdir -p gpurun_out
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2al_$TAG.json 2> gpurun_out/r2al_$TAG.err; echo "$TAG rc=$?"; }
TAG=d3 run
RSV_LIB=$PWD/tools/_rsv_d2.so TAG=d2 run
TAG=d3b run
RSV_LIB=$PWD/tools/_rsv_d2.so TAG=d2b run
