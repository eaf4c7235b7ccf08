#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_behaviour_gpu.py tests/test_sharding_fused_gpu.py -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2c_pytest.log
timeout 600 python tools/stepprof.py 29 30 1 > gpurun_out/r2c_prof_regen.txt 2>&1; echo rc=$?
timeout 600 python tools/stepprof.py 29 30 0 > gpurun_out/r2c_prof_split.txt 2>&1; echo rc=$?
tail -1 gpurun_out/r2c_prof_regen.txt; tail -1 gpurun_out/r2c_prof_split.txt
timeout 600 python bench.py --workload lattice20 --qubits 20 --steps 297 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2c_l20.json 2> gpurun_out/r2c_l20.err; echo "l20 rc=$?"
