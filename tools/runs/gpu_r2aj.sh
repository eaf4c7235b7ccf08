#!/bin/bash
# lo pass with 256 threads x 16 amplitudes (4 register bits) vs 512 x 8 (default), N=29 pulse; parity first
mkdir -p gpurun_out
RSV_LIB=$PWD/tools/_rsv_lo256.so timeout 900 python -m pytest tests/test_headline_parity_gpu.py tests/test_gpu_parity.py -q -x -k "multi_pass or plan or N29 or n29 or whole" > gpurun_out/r2aj_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2aj_pytest.log
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2aj_$TAG.json 2> gpurun_out/r2aj_$TAG.err; echo "$TAG rc=$?"; }
TAG=lo512 run
RSV_LIB=$PWD/tools/_rsv_lo256.so TAG=lo256 run
TAG=lo512b run
RSV_LIB=$PWD/tools/_rsv_lo256.so TAG=lo256b run
