#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_reference_behaviour_gpu.py -q -x > gpurun_out/r2ad_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ad_pytest.log
run() { timeout 600 python bench.py --workload lattice20 --qubits 20 --steps 297 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2ad_$TAG.json 2> gpurun_out/r2ad_$TAG.err; echo "$TAG rc=$?"; }
TAG=pf run
RSV_LIB=$PWD/tools/_rsv_nopf.so TAG=nopf run
TAG=pf2 run
RSV_LIB=$PWD/tools/_rsv_nopf.so TAG=nopf2 run
