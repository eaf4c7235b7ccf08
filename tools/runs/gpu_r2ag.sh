#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2ag_bench.json 2> gpurun_out/r2ag_bench.err; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_headline_parity_gpu.py tests/test_gpu_parity.py -q -x -k "full or max or N29 or n29 or expm" > gpurun_out/r2ag_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2ag_pytest.log
