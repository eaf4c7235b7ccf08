#!/bin/bash
# mid pass on the rotating-buffer body (operand one tile ahead, TMA-store output) vs the TMA body
mkdir -p gpurun_out
RSV_LIB=$PWD/tools/_rsv_rotmid.so timeout 900 python -m pytest tests/test_headline_parity_gpu.py tests/test_gpu_parity.py -q -x -k "whole or steps or multi_pass" > gpurun_out/r2ao_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ao_pytest.log
run() { timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/r2ao_$TAG.json 2> gpurun_out/r2ao_$TAG.err; echo "$TAG rc=$?"; }
TAG=def run
RSV_LIB=$PWD/tools/_rsv_rotmid.so TAG=rot run
TAG=def2 run
RSV_LIB=$PWD/tools/_rsv_rotmid.so TAG=rot2 run
