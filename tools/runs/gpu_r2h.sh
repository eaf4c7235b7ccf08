#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharding_fused_gpu.py tests/test_gpu_parity.py -x -q -k "not full_sweep" > gpurun_out/r2h_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2h_pytest.log
bash tools/ncu_capture.sh r2h 29
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2h_launches.log 2>&1; echo "launches rc=$?"
