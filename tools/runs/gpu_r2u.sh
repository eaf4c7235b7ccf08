#!/bin/bash
# peer-memory TMA ring: sharded tests (2/4 ranks on one GPU through CUDA IPC), then the N=28 full-size case
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_sharding_fused_gpu.py -q -x > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r2u_pytest.log
