#!/bin/bash
# mid pass at 128 threads x 32 amplitudes (5 register bits, two output halves) vs 256 x 16: parity, then A/B
mkdir -p gpurun_out
RSV_LIB=$PWD/tools/_rsv_mid128.so timeout 1200 python -m pytest tests/test_headline_parity_gpu.py tests/test_gpu_parity.py tests/test_sharding_fused_gpu.py -q -x > gpurun_out/r2am_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2am_pytest.log
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2am_$TAG.json 2> gpurun_out/r2am_$TAG.err; echo "$TAG rc=$?"; }
TAG=m256 run
RSV_LIB=$PWD/tools/_rsv_mid128.so TAG=m128 run
TAG=m256b run
RSV_LIB=$PWD/tools/_rsv_mid128.so TAG=m128b run
