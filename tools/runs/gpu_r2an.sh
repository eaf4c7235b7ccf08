#!/bin/bash
# N=29: the 9-bit group in the last pass (a=3) and the 8-bit group in the mid pass (a=4) vs the default
mkdir -p gpurun_out
RSV_LIB=$PWD/tools/_rsv_topbig.so timeout 900 python -m pytest tests/test_headline_parity_gpu.py -q -x > gpurun_out/r2an_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2an_pytest.log
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2an_$TAG.json 2> gpurun_out/r2an_$TAG.err; echo "$TAG rc=$?"; }
TAG=def run
RSV_LIB=$PWD/tools/_rsv_topbig.so TAG=top run
TAG=def2 run
RSV_LIB=$PWD/tools/_rsv_topbig.so TAG=top2 run
