#!/bin/bash
# lane-bit flips by warp shuffles: parity, then A/B bench (N=29 pulse) against the LDS build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity_gpu.py -q -x > gpurun_out/r2ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ab_pytest.log
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2ab_$TAG.json 2> gpurun_out/r2ab_$TAG.err; echo "$TAG rc=$?"; }
TAG=shfl run
RSV_LIB=$PWD/tools/_rsv_noshfl.so TAG=lds run
TAG=shfl2 run
RSV_LIB=$PWD/tools/_rsv_noshfl.so TAG=lds2 run
