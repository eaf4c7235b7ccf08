#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -k "not full_sweep" > gpurun_out/r2f_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2f_pytest.log
timeout 900 python bench.py --no-cpu > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload lattice20 --qubits 20 --steps 297 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2f_l20.json 2> gpurun_out/r2f_l20.err; echo "l20 rc=$?"
